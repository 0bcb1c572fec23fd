"""One oz2_dgemm call for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    python tools/sanitize_case.py M N K NMOD CG FUSED [scheme] [mode] [transa transb] [tile_n]

CG = OZ2_TUNE_CTA_GROUP (1, 2, 4), FUSED = OZ2_TUNE_FUSED_CRT (0 / 1); host inputs (numpy),
device buffers, every stage enabled; prints the residue of C against a cuBLAS DGEMM as a
sanity check (the sanitizer's own verdict is the point)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_host

m, n, k, N, cg, fused = (int(x) for x in sys.argv[1:7])
scheme = sys.argv[7] if len(sys.argv) > 7 else "fp8"
mode = sys.argv[8] if len(sys.argv) > 8 else "accurate"
transa, transb = (sys.argv[9], sys.argv[10]) if len(sys.argv) > 10 else ("N", "N")
tile_n = int(sys.argv[11]) if len(sys.argv) > 11 else 256
Ah = torch.from_numpy(gen_host(m, k, "phi", phi=1.0, seed=1)).cuda()
Bh = torch.from_numpy(gen_host(k, n, "phi", phi=1.0, seed=2)).cuda()
# column-major storage of op(A) (m x k, lda = m) or of A^T (k x m, lda = k); same for B
A, lda = (Ah.t().contiguous().t(), m) if transa == "N" else (Ah.contiguous(), k)
B, ldb = (Bh.t().contiguous().t(), k) if transb == "N" else (Bh.contiguous(), n)
C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
assert P.oz2_set_tuning("cta_group", cg) == 0 and P.oz2_set_tuning("fused_crt", fused) == 0
assert P.oz2_set_tuning("tile_n", tile_n) == 0
assert P.oz2_set_scheme(scheme) == 0 and P.oz2_set_mode(mode) == 0
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
rc = P.oz2_dgemm(transa, transb, m, n, k, 1.0, A.data_ptr(), lda, B.data_ptr(), ldb, 0.0, C.data_ptr(), m, N)
torch.cuda.synchronize()
ref = Ah @ Bh
print(f"case m={m} n={n} k={k} N={N} cg={cg} fused={fused} {scheme} {mode} {transa}{transb} tile_n={tile_n}: rc={rc} "
      f"rel={(torch.linalg.norm(C - ref) / torch.linalg.norm(ref)).item():.2e}", flush=True)
if rc != 0:
    print("last CUDA error:", P.oz2_last_cuda_error(), flush=True)
P.oz2_finalize()
sys.exit(0 if rc == 0 else 1)
