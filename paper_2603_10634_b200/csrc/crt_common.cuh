// crt_common.cuh -- exact per-element Chinese-remainder reconstruction and inverse
// scaling (eq. CRT_finalreduction, eq. inversescaling), shared by
// the standalone k_crt and the fused epilogue of the residue GEMM.
//
// With u_l = C'_l mod p_l in [0, p_l) (the residue GEMM stores u_l) and w_l = q_l P/p_l:
//   S = sum_l u_l w_l                     (exact, L 32-bit limbs, wrap-around mod 2^(32L))
//   t = round(sum_l u_l q_l/p_l)          (fixed point, 2^-32 units: S/P to within 2^-19)
//   C' = S - t P  (mod 2^(32L)), then one correction into [-P/2, P/2)   (symmetric, R2)
// 2^(32L-1) > 1.5 P, so the two's-complement value of the L-limb result is exact even
// when t is off by one (|frac(S/P) - 1/2| < 2^-19), and one correction fixes that case.
// RN64(|C'|) from the top 64 significant bits with a sticky bit (exact RNE), then an
// exact power-of-two scaling by 2^-(e_mu_i + e_nu_j) (exact unless subnormal, R10).
#pragma once
#include <cstdint>
#include "oz2_internal.h"

namespace oz2 {

template <int L>
__device__ __forceinline__ int cmp_limbs(const uint32_t (&a)[L], const uint32_t* b) {
#pragma unroll
    for (int t = L - 1; t >= 0; --t) {
        if (a[t] != b[t]) return a[t] > b[t] ? 1 : -1;
    }
    return 0;
}

template <int L>
__device__ __forceinline__ void add_limbs(uint32_t (&a)[L], const uint32_t* b) {
    uint64_t c = 0;
#pragma unroll
    for (int t = 0; t < L; ++t) {
        const uint64_t s = static_cast<uint64_t>(a[t]) + b[t] + c;
        a[t] = static_cast<uint32_t>(s);
        c = s >> 32;
    }
}

template <int L>
__device__ __forceinline__ void negate_limbs(uint32_t (&a)[L]) {
    uint64_t c = 1;
#pragma unroll
    for (int t = 0; t < L; ++t) {
        const uint64_t s = static_cast<uint64_t>(~a[t]) + c;
        a[t] = static_cast<uint32_t>(s);
        c = s >> 32;
    }
}

// constants of one plan staged in shared memory (broadcast reads)
struct CrtShared {
    uint32_t w[kMaxModuli][kMaxLimbs];
    uint32_t qp[kMaxModuli];
    uint32_t p[kMaxModuli];
};

__device__ __forceinline__ void crt_stage_constants(CrtShared* s, const CrtParams& cp, int tid, int nthreads) {
    for (int t = tid; t < cp.num_moduli * kMaxLimbs; t += nthreads) s->w[t / kMaxLimbs][t % kMaxLimbs] = cp.w[t / kMaxLimbs][t % kMaxLimbs];
    for (int t = tid; t < cp.num_moduli; t += nthreads) {
        s->qp[t] = cp.qp32[t];
        s->p[t] = static_cast<uint32_t>(cp.p[t]);
    }
}

template <int L>
__device__ __forceinline__ double crt_finish(const uint64_t (&acc)[L], uint64_t tacc, const CrtParams& cp,
                                             int escale);

// value of C'(i,j) * 2^-escale, rounded once to nearest binary64; rp points at the
// residue of modulus 0 of the element, residues of modulus l at rp + l * lstride
template <int L>
__device__ __forceinline__ double crt_element(const int16_t* rp, int64_t lstride, const CrtShared* s,
                                              const CrtParams& cp, int escale, bool streaming) {
    const int nm = cp.num_moduli;
    uint64_t acc[L];
#pragma unroll
    for (int t = 0; t < L; ++t) acc[t] = 0;
    uint64_t tacc = 0x80000000ull;                       // + 1/2: round-to-nearest of S/P
#pragma unroll 4
    for (int l = 0; l < nm; ++l) {
        const uint16_t* up = reinterpret_cast<const uint16_t*>(rp + l * lstride);   // u_l in [0, p_l)
        const uint32_t u = streaming ? static_cast<uint32_t>(__ldcs(up)) : static_cast<uint32_t>(__ldg(up));
        tacc += static_cast<uint64_t>(u) * s->qp[l];    // sum u_l q_l/p_l in 2^-32 units
#pragma unroll
        for (int t = 0; t < L; ++t) acc[t] += static_cast<uint64_t>(u) * s->w[l][t];
    }
    return crt_finish<L>(acc, tacc, cp, escale);
}

// rare path of crt_finish: the quotient estimate was off by one, C' outside [-P/2, P/2)
template <int L>
__device__ __noinline__ void crt_fix_range(uint32_t (&r)[L], const CrtParams& cp) {
    if ((r[L - 1] >> 31) == 0u) {
        if (cmp_limbs<L>(r, cp.halfP) >= 0) add_limbs<L>(r, cp.np);    // C' >= P/2: subtract P
    } else {
        uint32_t a[L];
#pragma unroll
        for (int t = 0; t < L; ++t) a[t] = r[t];
        negate_limbs<L>(a);
        if (cmp_limbs<L>(a, cp.halfP) > 0) add_limbs<L>(r, cp.P);       // C' < -P/2: add P
    }
}

// the rest of the reconstruction from the accumulated S (L limbs of 64-bit partial sums)
// and the fixed-point quotient estimate; branch-free on the common path
template <int L>
__device__ __forceinline__ double crt_finish(const uint64_t (&acc)[L], uint64_t tacc, const CrtParams& cp,
                                             int escale) {
    const uint32_t tq = static_cast<uint32_t>(tacc >> 32);   // t = round(S / P) (+-1)
    uint32_t r[L];
    uint64_t carry = 0;
#pragma unroll
    for (int t = 0; t < L; ++t) {
        const uint64_t v = acc[t] + static_cast<uint64_t>(tq) * cp.np[t] + carry;
        r[t] = static_cast<uint32_t>(v);
        carry = v >> 32;
    }
    // with T the signed top limb and H_top that of P/2, -H_top <= T < H_top already puts C'
    // in [-P/2, P/2) (the quotient estimate is almost never off by one)
    {
        const int T = static_cast<int>(r[L - 1]);
        const int Ht = static_cast<int>(cp.halfP[L - 1]);
        if (T >= Ht || T < -Ht) crt_fix_range<L>(r, cp);
    }
    // |C'| in two's complement, branch-free: r ^= s, r += (s & 1) with s the sign mask
    const uint32_t sm = static_cast<uint32_t>(static_cast<int>(r[L - 1]) >> 31);
    const bool negv = sm != 0u;
    {
        uint64_t c = sm & 1u;
#pragma unroll
        for (int t = 0; t < L; ++t) {
            const uint64_t v = static_cast<uint64_t>(r[t] ^ sm) + c;
            r[t] = static_cast<uint32_t>(v);
            c = v >> 32;
        }
    }
    // 64-bit words, the top nonzero one found by selects
    constexpr int NW = (L + 1) / 2;
    uint64_t w[NW];
#pragma unroll
    for (int q = 0; q < NW; ++q)
        w[q] = static_cast<uint64_t>(r[2 * q]) | (2 * q + 1 < L ? static_cast<uint64_t>(r[2 * q + 1]) << 32 : 0ull);
    uint64_t hiw = w[0], low = 0, below = 0;
    int tp = 0;
#pragma unroll
    for (int q = 1; q < NW; ++q) {
        if (w[q] != 0ull) {                   // predicated selects (unrolled, no divergence)
            tp = q;
            hiw = w[q];
            low = w[q - 1];
            uint64_t o = 0;
#pragma unroll
            for (int u = 0; u + 1 < q; ++u) o |= w[u];
            below = o;
        }
    }
    double v;
    int ex;
    if (tp == 0) {
        v = __ull2double_rn(hiw);             // exact RNE of |C'| < 2^64
        ex = 0;
    } else {
        const int lz = __clzll(static_cast<long long>(hiw));
        const uint64_t top64 = lz ? (hiw << lz) | (low >> (64 - lz)) : hiw;
        const bool sticky = (lz ? ((low << lz) != 0ull) : (low != 0ull)) || below != 0ull;
        v = __ull2double_rn(top64 | (sticky ? 1ull : 0ull));   // RNE from 64 bits + sticky
        ex = 64 * tp - lz;                                     // |C'| ~ top64 * 2^ex
    }
    const int E = ex - escale;
    if (v != 0.0 && E >= -1022 && E <= 1023 - 64)
        v *= __longlong_as_double(static_cast<long long>(E + 1023) << 52);
    else if (v != 0.0)
        v = ldexp(v, E);
    return negv ? -v : v;
}

// inverse-scaling exponent of element (i, j), or the NaN marker when row i of op(A) or
// column j of op(B) held a NaN / Inf (R12)
__device__ __forceinline__ bool exps_finite(int emu, int enu) {
    return emu != kExpNonFinite && enu != kExpNonFinite;
}

// C <- alpha v + beta C (R11; beta == 0 never reads C)
__device__ __forceinline__ void store_alpha_beta(double* cptr, double v, double alpha, double beta) {
    if (beta == 0.0) *cptr = alpha * v;
    else *cptr = fma(alpha, v, beta * *cptr);
}

}  // namespace oz2
