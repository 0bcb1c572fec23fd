"""Quick timing of the pipeline (development aid, not the bench contract)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device


def time_call(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts), sorted(ts)[len(ts) // 2]


def main():
    sizes = [int(x) for x in (sys.argv[1:] or ["4096", "8192", "16384"])]
    for n in sizes:
        for N in [12, 13]:
            A = gen_device(n, n, "phi", phi=1.0, seed=1)
            B = gen_device(n, n, "phi", phi=1.0, seed=2)
            C = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
            ws = torch.empty(P.oz2_workspace_size("N", "N", n, n, n, N), dtype=torch.uint8, device="cuda")
            P.oz2_set_workspace(ws.data_ptr(), ws.numel())
            P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)

            def f():
                rc = P.oz2_dgemm("N", "N", n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0,
                                 C.data_ptr(), n, N)
                assert rc == 0, rc
            tmin, tmed = time_call(f)
            flops = 2.0 * n ** 3
            fp8 = (3 * N + 1) * flops
            print(f"n={n} N={N}: {tmed:.2f} ms  emulated {flops / tmed / 1e9:.1f} TFLOP/s  "
                  f"FP8 {fp8 / tmed / 1e9:.0f} TFLOP/s", flush=True)
            ref = A @ B
            torch.cuda.synchronize()
            tn = time_call(lambda: A @ B)[1]
            err = (torch.linalg.norm(C - ref) / torch.linalg.norm(ref)).item()
            print(f"   cuBLAS dgemm {tn:.2f} ms = {flops / tn / 1e9:.1f} TFLOP/s;  |oz2 - dgemm|/|dgemm| = {err:.2e}",
                  flush=True)
            del A, B, C, ws, ref
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
