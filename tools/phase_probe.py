"""Per-phase CUDA-event timers of oz2_dgemm at one shape (medians over `reps` calls).

    python tools/phase_probe.py M N K NMOD [reps]
"""
import statistics
import sys
import torch
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device

m, n, k, N = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
A = gen_device(m, k, "phi", phi=1.0, seed=1)
B = gen_device(k, n, "phi", phi=1.0, seed=2)
C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
P.oz2_set_timing(True)
acc = {}
for r in range(reps + 3):
    assert P.oz2_dgemm("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0, C.data_ptr(), m, N) == 0
    t = P.oz2_get_timing()
    if r >= 3:
        for key, v in t.items():
            acc.setdefault(key, []).append(v)
ph = {key: round(statistics.median(v), 3) for key, v in acc.items()}
print(f"{m}x{n}x{k} N={N}: {2.0*m*n*k/ph['total']/1e9:.2f} TFLOP/s", ph, flush=True)
