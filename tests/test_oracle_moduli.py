"""Pins for oracle.moduli against the paper's printed lists and bounds."""
import math
import random
from fractions import Fraction

import pytest

from oracle import moduli as mod
from oracle import models


def test_prefixes(facts):
    for key, fn in [("int8_moduli_prefix", mod.int8_moduli),
                    ("karatsuba_moduli_prefix", mod.karatsuba_moduli),
                    ("hybrid_moduli_prefix", mod.hybrid_moduli)]:
        want = facts[key]["values"]
        assert fn(len(want)) == want, facts[key]["cite"]


def _log2(x):
    return mod.log2_big(x, 40)


def _prod(xs):
    P = 1
    for x in xs:
        P *= x
    return P


def test_thresholds(facts):
    fam = {"int8": mod.int8_moduli, "karatsuba": mod.karatsuba_moduli, "hybrid": mod.hybrid_moduli}
    for t in facts["thresholds"]:
        P = _prod(fam[t["family"]](t["N"]))
        assert P // 2 > 2 ** t["half_P_above_log2"] or (P % 2 == 1 and Fraction(P, 2) > 2 ** t["half_P_above_log2"]), t
        # and one fewer modulus does not reach it (why the paper needs exactly that N)
        P1 = _prod(fam[t["family"]](t["N"] - 1))
        assert Fraction(P1, 2) < 2 ** t["half_P_above_log2"], t


def _full_family(name):
    if name == "int8":
        return _greedy_all(256, [])
    if name == "karatsuba":
        return _greedy_all(513, [])
    sq = mod.hybrid_squares()
    return sq + _greedy_all(513, sq)


def _greedy_all(start, kept):
    kept = list(kept)
    out = []
    for c in range(start, 1, -1):
        if all(math.gcd(c, q) == 1 for q in kept):
            kept.append(c)
            out.append(c)
    return out


def test_family_bounds(facts):
    for fb in facts["family_bounds"]:
        full = _full_family(fb["family"])
        P = _prod(full)
        assert Fraction(P, 2) < 2 ** fb["half_P_full_below_log2"], fb
        first = full[0]
        if "half_P_N1_at_least_log2" in fb:
            assert Fraction(first, 2) >= 2 ** fb["half_P_N1_at_least_log2"]
        else:
            assert Fraction(first, 2) > 2 ** fb["half_P_N1_above_log2"]


def test_direct_fp8_set_too_small(facts):
    d = facts["direct_fp8_moduli"]
    assert all(math.gcd(a, b) == 1 for i, a in enumerate(d["values"]) for b in d["values"][i + 1:])
    assert Fraction(_prod(d["values"]), 2) < 2 ** d["half_P_below_log2"]


def test_six_squares_and_seventh_at_34(facts):
    sq = mod.hybrid_squares()
    assert len(sq) == facts["n_squares_assumed"]["n_squares"]
    lst = mod.hybrid_squares() + _greedy_all(513, sq)
    # the first further perfect square in the list sits at 1-based index N_limit
    idx = next(i for i, p in enumerate(lst) if i >= 6 and mod.is_square(p))
    assert idx + 1 == facts["n_squares_assumed"]["N_limit"]
    assert lst[idx] == 19 * 19


def test_pairwise_coprime_and_square_flags():
    for N in range(2, 34):
        ps = mod.hybrid_moduli(N)
        assert all(math.gcd(a, b) == 1 for i, a in enumerate(ps) for b in ps[i + 1:])
        for i, p in enumerate(ps):
            assert mod.is_square(p) == (i < 6)
            if i >= 6:
                assert p <= 513
            else:
                assert math.isqrt(p) <= 33


def test_crt_weights_identity(spec):
    for ps, P, w in spec["crt"]["plans"]:
        plan = mod.crt_plan(ps)
        assert plan.P == P and list(plan.w) == w
    for N in [2, 6, 12, 13, 14, 20, 33]:
        plan = mod.crt_plan(mod.hybrid_moduli(N))
        for l, w in enumerate(plan.w):
            for j, p in enumerate(plan.moduli):
                assert w % p == (1 if j == l else 0)


def test_crt_round_trip():
    rnd = random.Random(5)
    for N in [2, 12, 13, 20]:
        plan = mod.crt_plan(mod.hybrid_moduli(N))
        for _ in range(300):
            x = rnd.randrange(-(plan.P // 2), plan.P // 2)
            r = [mod.smod(x, p) for p in plan.moduli]
            y = mod.smod(sum(w * c for w, c in zip(plan.w, r)), plan.P)
            assert y == x


def test_crt_brute_force_small(spec):
    ps, res, want = spec["crt"]["reconstruct"]
    plan = mod.crt_plan(ps)
    got = mod.smod(sum(w * c for w, c in zip(plan.w, res)), plan.P)
    # brute force over the symmetric range
    bf = [x for x in range(-plan.P // 2, plan.P // 2) if x % ps[0] == res[0] % ps[0] and x % ps[1] == res[1] % ps[1]]
    assert bf == [want] and got == want


def test_smod(spec):
    for x, p, r in spec["smod"]["cases"]:
        assert mod.smod(x, p) == r
    for p in [7, 8, 255, 256, 1024, 1089]:
        vals = sorted({mod.smod(x, p) for x in range(-3 * p, 3 * p)})
        assert len(vals) == p and vals[-1] - vals[0] == p - 1
        assert vals[0] == -(p // 2)


def test_log2_big_and_pprime():
    for x in [2, 3, 10 ** 30 + 7, 2 ** 200 - 1]:
        v = mod.log2_big(x, 60)
        assert abs(float(v) - math.log2(x)) < 1e-12
        assert Fraction(2) ** 0 <= Fraction(x, 2 ** math.floor(v))   # sanity
    for N in [12, 13, 14]:
        P = _prod(mod.hybrid_moduli(N))
        Pp = mod.p_prime(P)
        true = (math.log2(P - 1) - 1) / 2
        assert float(Pp) <= true and true - float(Pp) < 2 ** -18 * 64


def test_table2(facts):
    for row in facts["table2"]["rows"]:
        assert models.matmul_count(row["method"], "fast", row["param"]) == row["fast"]
        assert models.matmul_count(row["method"], "accurate", row["param"]) == row["accurate"]
        if row["method"] == "fp8-ozaki1":
            assert 5 * row["param"] - 1 == row["bits_le"]
        else:
            fam = mod.hybrid_moduli if row["method"] == "fp8-ozaki2" else mod.int8_moduli
            assert math.floor(mod.effective_bits(fam(row["param"]))) == row["bits_le"]
    S = facts["ozaki1_bits"]["S_min"]
    assert 5 * S - 1 >= 53 > 5 * (S - 1) - 1


def test_M_N_and_workspace(facts):
    for N, M in facts["M_N"]["pairs"]:
        assert models.M_N(N) == M
    # M_N counts the digit planes: 2 per square modulus, 3 per non-square
    for N in range(1, 34):
        assert models.M_N(N) == 2 * min(N, 6) + 3 * max(N - 6, 0)
    w = facts["workspace"]
    # the paper quotes the byte counts rounded up to whole GB (26.3 -> 27, 54.8 -> 55)
    assert math.ceil(models.workspace_i8(16384, 16384, 16384, 14) / 1e9) == w["W_i8_16384_N14_GB"]
    assert math.ceil(models.workspace_f8(16384, 16384, 16384, 12) / 1e9) == w["W_f8_16384_N12_GB"]
