"""Run the pipeline a few times at one size (for ncu launch lists / captures).

    python tools/profile_once.py [n] [N] [reps] [scheme] [mode] ["knob=v,knob=v"]
"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
N = int(sys.argv[2]) if len(sys.argv) > 2 else 13
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
scheme = sys.argv[4] if len(sys.argv) > 4 else "fp8"
mode = sys.argv[5] if len(sys.argv) > 5 else "accurate"
knobs = sys.argv[6] if len(sys.argv) > 6 else ""     # "knob=v,knob=v" (oz2_set_tuning)
for kv in filter(None, knobs.split(",")):
    kn, v = kv.split("=")
    assert P.oz2_set_tuning(kn, int(v)) == 0, kv
A = gen_device(n, n, "phi", phi=1.0, seed=1)
B = gen_device(n, n, "phi", phi=1.0, seed=2)
C = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
assert P.oz2_set_scheme(scheme) == 0 and P.oz2_set_mode(mode) == 0
ws = torch.empty(P.oz2_workspace_size("N", "N", n, n, n, N), dtype=torch.uint8, device="cuda")
P.oz2_set_workspace(ws.data_ptr(), ws.numel())
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
P.oz2_set_timing(True)
for _ in range(reps):
    assert P.oz2_dgemm("N", "N", n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0, C.data_ptr(), n, N) == 0
    print({k: round(v, 3) for k, v in P.oz2_get_timing().items()}, flush=True)
torch.cuda.synchronize()
