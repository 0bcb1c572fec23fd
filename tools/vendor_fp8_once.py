"""cuBLASLt FP8 GEMM (torch._scaled_mm, e4m3, 16384^3, digits-like data) a few times,
for an ncu capture beside the residue GEMM (same box, same data class)."""
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
torch.cuda.synchronize()
print("ok")
