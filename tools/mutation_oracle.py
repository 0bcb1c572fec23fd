"""Mutation check of the oracle's pins: apply one plausible mistake at a time to a temp
copy of oracle/ and run the -m "not gpu" oracle tests; a mutation that survives marks an
unpinned spot.  python tools/mutation_oracle.py"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTATIONS = [
    ("scheme.py", "return fp32.round_down(Fraction(math.log2(float(c))))",
     "return fp32.round_nearest(Fraction(math.log2(float(c))))", "log2_rd32 RN"),
    ("moduli.py", "    return r\n\n\ndef delta", "    return r - 8 * Fraction(1, 2 ** 18)\n\n\ndef delta", "P' -8 ulp"),
    ("scheme.py", "return fp32.round_up(Fraction(1) / (1 - Fraction(k, 2 ** 23)))",
     "return 4 * fp32.round_up(Fraction(1) / (1 - Fraction(k, 2 ** 23)))", "f_k x4"),
    ("scheme.py", "        e = 7 - ufp_exp(mx)", "        e = 8 - ufp_exp(mx)", "prescale 7 -> 8"),
    ("scheme.py", "    x3 = fp32.round_down(Pp + x2)", "    x3 = fp32.round_up(Pp + x2)", "offset RU"),
    ("scheme.py", "    return math.floor(x3)", "    return math.ceil(x3)", "int() ceil"),
    ("scheme.py", "    cbar = fp32.round_up(safety_factor(k) * Rmax)", "    cbar = fp32.round_down(safety_factor(k) * Rmax)", "cbar RD"),
    ("scheme.py", "    d1 = round(Fraction(r, s))", "    d1 = math.floor(Fraction(r, s) + Fraction(1, 2))", "square digit ties up"),
    ("scheme.py", "    d1 = (a + 15) // 16", "    d1 = (a + 8) // 16", "karatsuba ceil->round"),
    ("scheme.py", "    return f(256 * C1 + C2 + 16 * (C3 - C1 - C2))", "    return f(256 * C1 + C2 + 16 * (C3 - C1 + C2))", "karatsuba sign"),
    ("scheme.py", "    return f(s * X.astype(object) + Y.astype(object))", "    return f(s * X.astype(object) - Y.astype(object))", "square combine sign"),
    ("scheme.py", "        q = abs(num) // den\n", "        q = (abs(num) + den - 1) // den\n", "to_integral ceil"),
    # (a strict first loop in fast_offset is an equivalent mutant: the second loop restores
    # the inclusive boundary; a dropped second loop or an off-by-one start is what can break)
    ("scheme.py", "    while Fraction(2) ** (2 * (t + 1)) * S <= H:\n        t += 1\n    return t",
     "    return t - 1", "fast offset off by one"),
    ("scheme.py", "    return round_down64(Fraction(plan.P - 1, 2))", "    return round_up64(Fraction(plan.P - 1, 2))", "fast H RU"),
    ("scheme.py", "            out[idx] = float(Fraction(alpha) * Fraction(x) + Fraction(bc))",
     "            out[idx] = float(Fraction(alpha) * Fraction(x) - Fraction(bc))", "alpha beta sign"),
    ("moduli.py", "    if 2 * r >= p:\n        r -= p", "    if 2 * r > p:\n        r -= p", "smod even range"),
    ("moduli.py", "    return fp32.round_down(Fraction(-1) / (2 - Fraction(1, 2 ** 21)))",
     "    return fp32.round_up(Fraction(-1) / (2 - Fraction(1, 2 ** 21)))", "delta RU"),
    ("fp8.py", None, None, "fp8 codec (skipped: exhaustive pins)"),
    ("int8.py", "        e = 6 - scheme.ufp_exp(mx)", "        e = 7 - scheme.ufp_exp(mx)", "int8 prescale 6 -> 7"),
    ("int8.py", "                bars[r, h] = math.ceil(abs(Fraction(v)) * scale)", "                bars[r, h] = round(abs(Fraction(v)) * scale)", "int8 bar ceil->round"),
    ("exact.py", "    e = ((ah * bh - p) + ah * bl + al * bh) + al * bl", "    e = ((ah * bh - p) + ah * bl + al * bh)", "TwoProduct dropped term"),
    ("exact.py", "            out[i, j] = (sb[j] * 2.0 ** (-e_mu[i]) + sa[i] * 2.0 ** (-e_nu[j])\n",
     "            out[i, j] = (sb[j] * 2.0 ** (-e_mu[i] - 1) + sa[i] * 2.0 ** (-e_nu[j] - 1)\n", "apriori bound halved"),
    ("scheme.py", "    return fp32.round_nearest(Fraction(int(exact_scaled), 2 ** 18))",
     "    return fp32.round_down(Fraction(int(exact_scaled), 2 ** 18))", "mma model RD"),
    ("scheme.py", "        acc = 0\n        for w, R in zip(plan.w, res_list):\n            acc += w * int(R[idx])",
     "        acc = 0\n        for w, R in zip(plan.w[::-1], res_list):\n            acc += w * int(R[idx])", "crt weight order"),
]


def main():
    tests = ["tests/test_oracle_pins.py", "tests/test_oracle_scheme.py", "tests/test_oracle_moduli.py",
             "tests/test_oracle_fp8_fp32.py", "tests/test_oracle_int8.py", "tests/test_sampled_helpers.py"]
    surv = []
    for fname, old, new, label in MUTATIONS:
        if old is None:
            continue
        tmp = tempfile.mkdtemp()
        for d in ["oracle", "synth", "tests"]:
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d))
        p = os.path.join(tmp, "oracle", fname)
        src = open(p).read()
        if old not in src:
            print(f"[skip] {label}: pattern not found")
            continue
        open(p, "w").write(src.replace(old, new, 1))
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider"] + tests,
                           cwd=tmp, capture_output=True, text=True, timeout=1800)
        killed = r.returncode != 0
        print(f"[{'killed' if killed else 'SURVIVED'}] {label}", flush=True)
        if not killed:
            surv.append(label)
        shutil.rmtree(tmp)
    print("survivors:", surv)
    return 1 if surv else 0


if __name__ == "__main__":
    sys.exit(main())
