"""Sustained throughput and SM clock under the power cap, back to back for `secs` seconds
each: (1) cuBLASLt FP8 (torch._scaled_mm) on digit-like data, (2) this repo's tcgen05 FP8
kernel on the SAME operands (oz2_fp8_gemm_raw: one product, FP32 out), (3) full oz2_dgemm
calls at 16384^3, N = 13 (39 residue products + conversions).  Separates the kernel's own
efficiency from the scheme's.

    python tools/power_probe.py [secs]
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from bench import ClockSampler
from synth import gen_device

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
n = 16384
g = torch.Generator(device="cuda")
g.manual_seed(5)
a8 = torch.randint(-16, 17, (n, n), generator=g, device="cuda").to(torch.float8_e4m3fn)
b8 = torch.randint(-16, 17, (n, n), generator=g, device="cuda").to(torch.float8_e4m3fn)
one = torch.ones((), dtype=torch.float32, device="cuda")
c32 = torch.empty((n, n), dtype=torch.float32, device="cuda")
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)


def sustained(name, f, flops):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s = ClockSampler(0)
    s.start()
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, t0 = 0, time.perf_counter()
    e0.record()
    while time.perf_counter() - t0 < secs:
        f()
        reps += 1
        if reps % 8 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = s.stop()
    out = {"name": name, "reps": reps, "tflops": round(flops * reps / (ms * 1e-3) / 1e12, 1),
           "sm_mhz": clk["sm_mhz"], "reasons": clk["reasons"]}
    print(json.dumps(out), flush=True)
    return out


res = []
res.append(sustained("cublaslt_fp8_scaled_mm", lambda: torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one,
                                                                         out_dtype=torch.bfloat16), 2.0 * n ** 3))
au, bu = a8.view(torch.uint8), b8.view(torch.uint8)
res.append(sustained("oz2_fp8_gemm_raw_same_data",
                     lambda: P.oz2_fp8_gemm_raw(au.data_ptr(), bu.data_ptr(), c32.data_ptr(), n, n, n), 2.0 * n ** 3))
# the same tcgen05 pipeline with step 2's near-empty epilogue (row / column maxima only)
rmax = torch.zeros(n, dtype=torch.int32, device="cuda")
smax = torch.zeros(n, dtype=torch.int32, device="cuda")
res.append(sustained("oz2_fp8_gemm_bound_same_data",
                     lambda: P.oz2_fp8_gemm_bound(au.data_ptr(), bu.data_ptr(), rmax.data_ptr(), smax.data_ptr(),
                                                  n, n, n), 2.0 * n ** 3))
res.append(sustained("cublaslt_fp8_scaled_mm_again", lambda: torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one,
                                                                               out_dtype=torch.bfloat16), 2.0 * n ** 3))
del a8, b8, c32
torch.cuda.empty_cache()
A = gen_device(n, n, "phi", phi=1.0, seed=1)
B = gen_device(n, n, "phi", phi=1.0, seed=2)
C = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
ws = torch.empty(P.oz2_workspace_size("N", "N", n, n, n, 13), dtype=torch.uint8, device="cuda")
P.oz2_set_workspace(ws.data_ptr(), ws.numel())
res.append(sustained("oz2_dgemm_N13_residue_products",
                     lambda: P.oz2_dgemm("N", "N", n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0,
                                         C.data_ptr(), n, 13), 39 * 2.0 * n ** 3))
