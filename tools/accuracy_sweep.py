"""Accuracy vs moduli count (BASELINE metric, second half) at the paper's shapes.

    python tools/accuracy_sweep.py [--size 16384] [--phis 0.5,1,2,4] [--moduli 12,13,14,16]
                                   [--sample 64] [--out gpurun_out/accuracy.json]

For every phi (paper generator) the same inputs go through oz2_dgemm (FP8 scheme,
accurate and fast modes, hybrid and Karatsuba-only moduli; INT8 scheme) and cuBLAS DGEMM
(torch.matmul float64).  Errors are measured against the exact product on a random
sample x sample block of entries (RN64 of the exact dot product: Dekker TwoProduct +
math.fsum, independent of oracle/).  Time per call is reported beside the errors.
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_10634_b200 as P  # noqa: E402
from synth import gen_device  # noqa: E402


def exact_block(Ah, Bh):
    """RN64 of the exact dot products Ah[a] . Bh[:, b] (TwoProduct + fsum)."""
    c = 134217729.0
    out = np.zeros((Ah.shape[0], Bh.shape[1]))
    bh_ = c * Bh
    bh = bh_ - (bh_ - Bh)
    bl = Bh - bh
    for a in range(Ah.shape[0]):
        x = Ah[a][:, None]
        xh_ = c * x
        xh = xh_ - (xh_ - x)
        xl = x - xh
        p = x * Bh
        e = ((xh * bh - p) + xh * bl + xl * bh) + xl * bl
        for b in range(Bh.shape[1]):
            out[a, b] = math.fsum(np.concatenate([p[:, b], e[:, b]]).tolist())
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=16384)
    ap.add_argument("--k", type=int, default=0, help="k (default: size)")
    ap.add_argument("--phis", default="0.5,1,2,4")
    ap.add_argument("--moduli", default="12,13,14,16")
    ap.add_argument("--sample", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/accuracy.json")
    a = ap.parse_args()
    m = n = a.size
    k = a.k or a.size
    Ns = [int(x) for x in a.moduli.split(",")]
    rng = np.random.default_rng(0)
    I = np.sort(rng.choice(m, a.sample, replace=False))
    J = np.sort(rng.choice(n, a.sample, replace=False))
    st = torch.cuda.current_stream()
    P.oz2_set_stream(st.cuda_stream)
    wsz = 0
    for sch in ("fp8", "karatsuba", "int8"):
        P.oz2_set_scheme(sch)
        wsz = max(wsz, max(P.oz2_workspace_size("N", "N", m, n, k, NN) for NN in Ns + [16]))
    P.oz2_set_scheme("fp8")
    ws = torch.empty(wsz, dtype=torch.uint8, device="cuda")
    P.oz2_set_workspace(ws.data_ptr(), ws.numel())
    C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    results = {"size": [m, n, k], "sample": f"{a.sample} x {a.sample} entries (exact: TwoProduct + fsum)",
               "device": torch.cuda.get_device_name(), "phi": {}}
    for phi in [float(x) for x in a.phis.split(",")]:
        A = gen_device(m, k, "phi", phi=phi, seed=11)
        B = gen_device(k, n, "phi", phi=phi, seed=12)
        t0 = time.time()
        ex = exact_block(A[I, :].cpu().numpy(), B[:, J].cpu().numpy())
        t_exact = time.time() - t0

        def errs(Cs):
            d = Cs - ex
            return {"normwise": float(np.linalg.norm(d) / np.linalg.norm(ex)),
                    "max_rel": float(np.max(np.abs(d) / np.abs(ex)))}

        def timed(f):
            f()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.reps):
                f()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / a.reps

        row = {}
        ref = torch.empty_like(C)
        ms = timed(lambda: torch.matmul(A, B, out=ref))
        row["cublas_dgemm"] = {"ms": round(ms, 3), "tflops": round(2.0 * m * n * k / ms / 1e9, 2),
                               **errs(ref[I][:, J].cpu().numpy())}
        for sch, mode, NNs in [("fp8", "accurate", Ns), ("fp8", "fast", Ns), ("karatsuba", "accurate", [13, 14]),
                               ("int8", "accurate", [14, 15, 16])]:
            P.oz2_set_scheme(sch)
            P.oz2_set_mode(mode)
            for NN in NNs:
                def f():
                    rc = P.oz2_dgemm("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0,
                                     C.data_ptr(), m, NN)
                    assert rc == 0, rc
                ms = timed(f)
                row[f"{sch}_{mode}_N{NN}"] = {"ms": round(ms, 3), "tflops": round(2.0 * m * n * k / ms / 1e9, 2),
                                              **errs(C[I][:, J].cpu().numpy())}
        P.oz2_set_scheme("fp8")
        P.oz2_set_mode("accurate")
        row["exact_seconds"] = round(t_exact, 1)
        results["phi"][str(phi)] = row
        print(json.dumps({str(phi): row}), flush=True)
        del A, B
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
