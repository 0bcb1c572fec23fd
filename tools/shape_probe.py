"""Time oz2_dgemm (device buffers, 10 calls after 5 warm-up) at one m, n, k, N."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device

m, n, k, N = (int(x) for x in sys.argv[1:5])
scheme = sys.argv[5] if len(sys.argv) > 5 else "fp8"
A = gen_device(m, k, "phi", phi=1.0, seed=1)
B = gen_device(k, n, "phi", phi=1.0, seed=2)
C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
assert P.oz2_set_scheme(scheme) == 0
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
f = lambda: P.oz2_dgemm("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0, C.data_ptr(), m, N)
for _ in range(5):
    assert f() == 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
ref = torch.matmul(A, B)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    torch.matmul(A, B, out=ref)
e1.record()
torch.cuda.synchronize()
msc = e0.elapsed_time(e1) / 5
print(f"{scheme} m={m} n={n} k={k} N={N}: {ms:.3f} ms = {2.0*m*n*k/ms/1e9:.2f} TFLOP/s; cuBLAS DGEMM {2.0*m*n*k/msc/1e9:.2f} TFLOP/s", flush=True)
