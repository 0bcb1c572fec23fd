// crt_kernel.cu -- Chinese-remainder reconstruction and inverse scaling
// (eq. CRT_finalreduction, eq. inversescaling).
//
// Per output element, with u_l = C'_l mod p_l in [0, p_l) and w_l = q_l P/p_l:
//   S = sum_l u_l w_l                     (exact, L 32-bit limbs, wrap-around mod 2^(32L))
//   t = round(sum_l u_l q_l/p_l)          (fixed point, 2^-32 units: S/P to within 2^-19)
//   C' = S - t P  (mod 2^(32L)), then one correction into [-P/2, P/2)   (symmetric, R2)
// 2^(32L-1) > 1.5 P, so the two's-complement value of the L-limb result is exact even
// when t is off by one (|frac(S/P) - 1/2| < 2^-19), and one correction fixes that case.
// C = RN64(C') * 2^-(e_mu_i + e_nu_j): the top 64 bits of |C'| with a sticky bit are
// rounded once to binary64 (exact RNE of C'), then scaled by a power of two (exact
// unless the result is subnormal, R10).  alpha/beta per R11.
#include <cstdint>
#include <cuda_runtime.h>
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

template <int L>
__global__ void __launch_bounds__(256) k_crt(const int16_t* __restrict__ res, int64_t m, int64_t n,
                                             const __grid_constant__ CrtParams cp,
                                             const int32_t* __restrict__ e_mu,
                                             const int32_t* __restrict__ e_nu, double alpha,
                                             double beta, double* __restrict__ C, int64_t ldc) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    if (i >= m) return;
    const int emu = e_mu[i];
    const int64_t lstride = n * m;
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
        uint64_t acc[L];
#pragma unroll
        for (int t = 0; t < L; ++t) acc[t] = 0;
        uint64_t tacc = 0x80000000ull;                  // + 1/2 for round-to-nearest of S/P
        const int16_t* rp = res + j * m + i;
#pragma unroll
        for (int l = 0; l < kMaxModuli; ++l) {     // static l: constants are direct operands
            if (l >= cp.num_moduli) break;
            const int c = __ldg(rp + l * lstride);
            const uint32_t u = static_cast<uint32_t>(c < 0 ? c + cp.p[l] : c);
            tacc += static_cast<uint64_t>(u) * cp.qp32[l];          // sum u_l q_l/p_l in 2^-32 units
#pragma unroll
            for (int t = 0; t < L; ++t) acc[t] += static_cast<uint64_t>(u) * cp.w[l][t];
        }
        const uint32_t tq = static_cast<uint32_t>(tacc >> 32);       // t = round(S / P) (+-1)
#pragma unroll
        for (int t = 0; t < L; ++t) acc[t] += static_cast<uint64_t>(tq) * cp.np[t];
        uint32_t r[L];
        uint64_t carry = 0;
#pragma unroll
        for (int t = 0; t < L; ++t) {
            const uint64_t v = acc[t] + carry;
            r[t] = static_cast<uint32_t>(v);
            carry = v >> 32;
        }
        // one correction into [-P/2, P/2)
        bool negv = (r[L - 1] >> 31) != 0;
        if (!negv) {
            if (cmp_limbs<L>(r, cp.halfP) >= 0) {             // C' >= P/2: subtract P
                add_limbs<L>(r, cp.np);
                negv = (r[L - 1] >> 31) != 0;
            }
        } else {
            uint32_t a[L];
#pragma unroll
            for (int t = 0; t < L; ++t) a[t] = r[t];
            negate_limbs<L>(a);
            if (cmp_limbs<L>(a, cp.halfP) > 0) {              // C' < -P/2: add P
                add_limbs<L>(r, cp.P);
                negv = (r[L - 1] >> 31) != 0;
            }
        }
        if (negv) negate_limbs<L>(r);
        // RNE(|C'|) via the top 64 significant bits + sticky (all limb indices static)
        uint32_t w2 = 0, w1 = r[1], w0 = r[0];
        int top = 1;
        bool sticky = false, found = false;
        uint32_t below = 0;                                  // OR of limbs under the window
#pragma unroll
        for (int t = L - 1; t >= 2; --t) {
            if (!found && r[t] != 0u) {
                found = true;
                top = t;
                w2 = r[t];
                w1 = r[t - 1];
                w0 = r[t - 2];
                uint32_t o = 0;
#pragma unroll
                for (int u = 0; u < t - 2; ++u) o |= r[u];
                below = o;
            }
        }
        double v;
        int ex;
        if (!found) {
            v = __ull2double_rn((static_cast<uint64_t>(w1) << 32) | w0);
            ex = 0;
        } else {
            const int lz = __clz(w2);
            const uint64_t hi = (static_cast<uint64_t>(w2) << 32) | w1;
            uint64_t top64 = lz ? (hi << lz) | (static_cast<uint64_t>(w0) >> (32 - lz)) : hi;
            sticky = (lz ? ((w0 << lz) != 0u) : (w0 != 0u)) || below != 0u;
            top64 |= sticky ? 1ull : 0ull;
            v = __ull2double_rn(top64);
            ex = 32 * (top - 1) - lz;                        // |C'| ~ top64 * 2^ex
        }
        const int E = ex - (emu + e_nu[j]);
        // v * 2^E exactly: one multiply by a constructed power of two when the result
        // stays normal (always, for sane inputs), ldexp otherwise
        if (v != 0.0 && E >= -1022 && E <= 1023 - 64)
            v *= __longlong_as_double(static_cast<long long>(E + 1023) << 52);
        else if (v != 0.0)
            v = ldexp(v, E);
        if (negv) v = -v;
        double* cptr = C + i + j * ldc;
        if (beta == 0.0) *cptr = alpha * v;
        else *cptr = fma(alpha, v, beta * *cptr);
    }
}

cudaError_t launch_crt(int limbs, const int16_t* res, int64_t m, int64_t n, const CrtParams& cp,
                       const int32_t* e_mu, const int32_t* e_nu, double alpha, double beta,
                       double* C, int64_t ldc, cudaStream_t st) {
    if (m == 0 || n == 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((m + 255) / 256), static_cast<unsigned>(n < 65535 ? n : 65535));
#define OZ2_CRT_CASE(LL) \
    case LL: k_crt<LL><<<grid, 256, 0, st>>>(res, m, n, cp, e_mu, e_nu, alpha, beta, C, ldc); break;
    switch (limbs) {
        OZ2_CRT_CASE(4)
        OZ2_CRT_CASE(5)
        OZ2_CRT_CASE(6)
        OZ2_CRT_CASE(7)
        OZ2_CRT_CASE(8)
        OZ2_CRT_CASE(9)
        OZ2_CRT_CASE(10)
        default: return cudaErrorInvalidValue;
    }
#undef OZ2_CRT_CASE
    return cudaGetLastError();
}

}  // namespace oz2
