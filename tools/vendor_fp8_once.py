"""cuBLASLt FP8 GEMM (torch._scaled_mm, e4m3, 16384^3, digits-like data) a few times,
for an ncu capture beside the residue GEMM (same box, same data class); with a third
argument `oz2`, also this repo's bound-mode tcgen05 GEMM (oz2_fp8_gemm_bound) on the same
operands."""
import sys
import torch
size = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device="cuda")
g.manual_seed(5)
a = torch.randint(-16, 17, (size, size), generator=g, device="cuda").to(torch.float8_e4m3fn)
b = torch.randint(-16, 17, (size, size), generator=g, device="cuda").to(torch.float8_e4m3fn)
one = torch.ones((), dtype=torch.float32, device="cuda")
for _ in range(reps):
    torch._scaled_mm(a, b.t(), scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
if len(sys.argv) > 3 and sys.argv[3] == "oz2":
    sys.path.insert(0, ".")
    import paper_2603_10634_b200 as P
    P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
    rmax = torch.zeros(size, dtype=torch.int32, device="cuda")
    smax = torch.zeros(size, dtype=torch.int32, device="cuda")
    au, bu = a.view(torch.uint8), b.view(torch.uint8)
    for _ in range(reps):
        assert P.oz2_fp8_gemm_bound(au.data_ptr(), bu.data_ptr(), rmax.data_ptr(), smax.data_ptr(),
                                    size, size, size) == 0
torch.cuda.synchronize()
print("ok")
