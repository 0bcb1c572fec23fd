"""The paper's throughput experiment: emulated DGEMM TFLOP/s vs k for square
m = n, FP8 Ozaki-II (accurate, N = 13) and INT8 Ozaki-II (accurate, N = 15) against native
cuBLAS DGEMM, one B200.  Each call is timed with CUDA events over `reps` calls after 3
warm-up calls; inputs are the paper generator with phi = 1.

    python tools/k_sweep.py [--mn 1024,2048,4096,8192,16384] [--k 1024,4096,16384,65536]
                            [--out gpurun_out/k_sweep.json]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_10634_b200 as P  # noqa: E402
from synth import gen_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mn", default="1024,2048,4096,8192,16384")
    ap.add_argument("--k", default="1024,4096,16384,65536")
    ap.add_argument("--out", default="gpurun_out/k_sweep.json")
    a = ap.parse_args()
    P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(f, flops):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        reps = max(3, min(50, int(2e13 / flops) + 1))      # ~0.2-1 s per point
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    rows = []
    for mn in [int(x) for x in a.mn.split(",")]:
        for k in [int(x) for x in a.k.split(",")]:
            if mn * k * 8 * 2 + mn * mn * 8 > 60e9:
                continue
            A = gen_device(mn, k, "phi", phi=1.0, seed=1)
            B = gen_device(k, mn, "phi", phi=1.0, seed=2)
            C = torch.empty((mn, mn), dtype=torch.float64, device="cuda").t()
            fl = 2.0 * mn * mn * k
            row = {"m": mn, "n": mn, "k": k}
            ms = timed(lambda: torch.matmul(A, B, out=C), fl)
            row["cublas_dgemm"] = round(fl / ms / 1e9, 2)
            for sch, N in [("fp8", 13), ("int8", 15)]:
                if sch == "int8" and k > 65536:
                    continue
                P.oz2_set_scheme(sch)

                def f():
                    rc = P.oz2_dgemm("N", "N", mn, mn, k, 1.0, A.data_ptr(), mn, B.data_ptr(), k, 0.0,
                                     C.data_ptr(), mn, N)
                    assert rc == 0, rc
                ms = timed(f, fl)
                row[f"oz2_{sch}_N{N}"] = round(fl / ms / 1e9, 2)
            P.oz2_set_scheme("fp8")
            P.oz2_finalize()
            rows.append(row)
            print(json.dumps(row), flush=True)
            del A, B, C
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump({"device": torch.cuda.get_device_name(), "phi": 1.0, "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
