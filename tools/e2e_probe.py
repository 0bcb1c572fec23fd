"""e2e time of oz2_dgemm on pinned host buffers at 16384^3 (N=13), vs the device-pointer call."""
import sys
import time
import torch
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
N = 13
A = gen_device(n, n, "phi", phi=1.0, seed=1)
B = gen_device(n, n, "phi", phi=1.0, seed=2)
Ah = torch.empty((n, n), dtype=torch.float64, pin_memory=True).t()
Bh = torch.empty((n, n), dtype=torch.float64, pin_memory=True).t()
Ch = torch.empty((n, n), dtype=torch.float64, pin_memory=True).t()
Ah.copy_(A)
Bh.copy_(B)
C = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    assert P.oz2_dgemm("N", "N", n, n, n, 1.0, Ah.data_ptr(), n, Bh.data_ptr(), n, 0.0, Ch.data_ptr(), n, N) == 0
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    assert P.oz2_dgemm("N", "N", n, n, n, 1.0, Ah.data_ptr(), n, Bh.data_ptr(), n, 0.0, Ch.data_ptr(), n, N) == 0
    ts.append(time.perf_counter() - t0)
assert P.oz2_dgemm("N", "N", n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0, C.data_ptr(), n, N) == 0
torch.cuda.synchronize()
same = torch.equal(C.cpu(), Ch)
e = min(ts)
print(f"e2e {e*1e3:.1f} ms = {2.0*n**3/e/1e12:.2f} TFLOP/s (min of 3), bit-identical to device call: {same}", flush=True)
