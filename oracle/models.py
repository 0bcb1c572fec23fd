"""Counting facts the build relies on (Sec. IV), written out from the paper.

* matmul counts: FP8 Ozaki-II 3N (fast) / 3N+1 (accurate), INT8 Ozaki-II N / N+1,
  FP8 Ozaki-I S(S+1)/2 / S^2 (Table 2).
* M_N = 2N (N <= 6) else 3N - 6 digit planes per operand (eq. M).
* workspace W_i8 = (mk + kn + 5mn)N + 2(m+n) (eq. W8i) and
  W_f8 = (mk + kn + 4mn)M_N + 2Nmn + 2(m+n) (eq. W8f).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""


def matmul_count(method: str, mode: str, param: int) -> int:
    if method == "fp8-ozaki2":
        return 3 * param + (1 if mode == "accurate" else 0)
    if method == "int8-ozaki2":
        return param + (1 if mode == "accurate" else 0)
    if method == "fp8-ozaki1":
        return param * param if mode == "accurate" else param * (param + 1) // 2
    raise ValueError(method)


def M_N(N: int) -> int:
    return 2 * N if N <= 6 else 3 * N - 6


def workspace_i8(m: int, n: int, k: int, N: int) -> int:
    return (m * k + k * n + 5 * m * n) * N + 2 * (m + n)


def workspace_f8(m: int, n: int, k: int, N: int) -> int:
    return (m * k + k * n + 4 * m * n) * M_N(N) + 2 * N * m * n + 2 * (m + n)
