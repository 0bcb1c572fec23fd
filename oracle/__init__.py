"""Oracle for the FP8 Ozaki-II DGEMM emulation (arxiv 2603.10634).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2603_10634_b200``) never imports it, and this
package never imports the product package: the two share no code.

What it is: a plain, slow, obviously-correct CPU implementation of what the paper
computes, written from PAPER.md (``P:n`` = PAPER.md line n).  Every function cites
the passage it follows.  Arithmetic is exact wherever the paper's result is exact:
Python integers for A', B', residues and the CRT (no fixed width), ``Fraction`` for
rational quantities and for the directed FP32 roundings of Sec. III-E, numpy int64
matmul (exact for |entries| <= 544, k <= 2^16) as the library primitive for the
integer residue products of eq. (CRTmatmul).

Modules
  fp8      E4M3 codec
  fp32     correctly directed rounding of rationals to binary32
  moduli   moduli families, P, q_l, CRT weights
  scheme   the emulation steps in the paper's order;
           FP8 families: hybrid (the method) and Karatsuba-only
  int8     the INT8 Ozaki-II baseline (bound and exponent rule: reading R16)
  exact    exact rational DGEMM references (for pins and accuracy metrics)
  models   matmul counts, M_N, workspace formulas (Table 2, eqs. M, W8i, W8f)

Every function here is pinned by a ``-m "not gpu"`` test against something other
than itself (paper-printed values, closed forms, brute force); see DESIGN.md
"Oracle pins".  There is no unpinned function.
"""
