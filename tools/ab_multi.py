"""A/B two sets of liboz2 tuning knobs in ONE process, alternating call by call.

    python tools/ab_multi.py SIZE N "knob=v,knob=v" "knob=v" [rounds] [k]

An empty set ("-") means the defaults.  Prints medians of the per-phase CUDA-event timers."""
import statistics
import sys
import torch
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device

n = int(sys.argv[1]); N = int(sys.argv[2]); sets = sys.argv[3:5]
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 8
k = int(sys.argv[6]) if len(sys.argv) > 6 else n
A = gen_device(n, k, "phi", phi=1.0, seed=1)
B = gen_device(k, n, "phi", phi=1.0, seed=2)
C = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
ws = torch.empty(P.oz2_workspace_size("N", "N", n, n, k, N), dtype=torch.uint8, device="cuda")
P.oz2_set_workspace(ws.data_ptr(), ws.numel())
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
P.oz2_set_timing(True)


def apply(spec):
    P.oz2_reset_tuning()
    if spec and spec != "-":
        for kv in spec.split(","):
            k, v = kv.split("=")
            assert P.oz2_set_tuning(k, int(v)) == 0, kv


res = {s: [] for s in sets}
for r in range(rounds + 1):
    for s in (sets if r % 2 == 0 else sets[::-1]):
        apply(s)
        assert P.oz2_dgemm("N", "N", n, n, k, 1.0, A.data_ptr(), n, B.data_ptr(), k, 0.0, C.data_ptr(), n, N) == 0
        t = P.oz2_get_timing()
        if r > 0:
            res[s].append(t)
for s in sets:
    tot = statistics.median(x["total"] for x in res[s])
    g = statistics.median(x["residue_gemm"] for x in res[s])
    ph = {key: round(statistics.median(x[key] for x in res[s]), 3) for key in res[s][0]}
    print(f"[{s}]: {2.0*n*n*k/tot/1e9:.2f} TFLOP/s", ph, flush=True)
