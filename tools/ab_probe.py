"""A/B a tuning knob of liboz2 (oz2_set_tuning, names in paper_2603_10634_b200.TUNE) in ONE
process, alternating settings call by call (so clock / power drift hits both arms alike).

    python tools/ab_probe.py SIZE N KNOB VAL_A VAL_B [rounds] [k] [scheme]
"""
import statistics
import sys
import torch
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device

n = int(sys.argv[1]); N = int(sys.argv[2]); var = sys.argv[3]; vals = sys.argv[4:6]
rounds = int(sys.argv[6]) if len(sys.argv) > 6 else 8
k = int(sys.argv[7]) if len(sys.argv) > 7 else n
scheme = sys.argv[8] if len(sys.argv) > 8 else "fp8"
m = n
A = gen_device(m, k, "phi", phi=1.0, seed=1)
B = gen_device(k, n, "phi", phi=1.0, seed=2)
C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
assert P.oz2_set_scheme(scheme) == 0
ws = torch.empty(P.oz2_workspace_size("N", "N", m, n, k, N), dtype=torch.uint8, device="cuda")
P.oz2_set_workspace(ws.data_ptr(), ws.numel())
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
P.oz2_set_timing(True)
res = {v: [] for v in vals}
for r in range(rounds + 1):
    for v in (vals if r % 2 == 0 else vals[::-1]):
        assert P.oz2_set_tuning(var, int(v)) == 0
        assert P.oz2_dgemm("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0, C.data_ptr(), m, N) == 0
        t = P.oz2_get_timing()
        if r > 0:
            res[v].append(t)
for v in vals:
    tot = statistics.median(x["total"] for x in res[v])
    g = statistics.median(x["residue_gemm"] for x in res[v])
    c = statistics.median(x["crt"] for x in res[v])
    ps = statistics.median(x["prescale"] for x in res[v])
    dg = statistics.median(x["digits"] for x in res[v])
    bg = statistics.median(x["bound_gemm"] for x in res[v])
    print(f"{var}={v}: total {tot:.3f} ms ({2.0*m*n*k/tot/1e9:.2f} TFLOP/s), residue_gemm {g:.3f}, "
          f"prescale {ps:.3f}, bound_gemm {bg:.3f}, digits {dg:.3f}, crt {c:.3f}", flush=True)
