// crt_kernel.cu -- Chinese-remainder reconstruction and inverse scaling
// (eq. CRT_finalreduction, eq. inversescaling).
//
// Per output element, with u_l = C'_l mod p_l in [0, p_l) and w_l = q_l P/p_l:
//   S = sum_l u_l w_l                     (exact, L 32-bit limbs, wrap-around mod 2^(32L))
//   t = rint(sum_l u_l q_l/p_l)           (FP64: S/P to within N 2^13 2^-53; t = round(S/P))
//   C' = S - t P  (mod 2^(32L)), then one correction into [-P/2, P/2)   (symmetric, R2)
// 2^(32L-1) > P, so the two's-complement value of the L-limb result is C' exactly.
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
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
        uint64_t acc[L];
#pragma unroll
        for (int t = 0; t < L; ++t) acc[t] = 0;
        double xq = 0.0;
        const int16_t* rp = res + j * m + i;
        const int64_t lstride = n * m;
#pragma unroll 1
        for (int l = 0; l < cp.num_moduli; ++l) {
            int c = rp[l * lstride];
            const int p = cp.p[l];
            const uint32_t u = static_cast<uint32_t>(c < 0 ? c + p : c);
            xq = fma(static_cast<double>(u), cp.qp[l], xq);
#pragma unroll
            for (int t = 0; t < L; ++t) acc[t] += static_cast<uint64_t>(u) * cp.w[l][t];
        }
        const uint32_t tq = static_cast<uint32_t>(rint(xq));
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
        // |C'| and its binary64 value (RNE) via the top 64 bits + sticky
        if (negv) negate_limbs<L>(r);
        int top = L - 1;
        while (top > 0 && r[top] == 0) --top;
        double v;
        if (top <= 1) {
            const uint64_t mag = (static_cast<uint64_t>(top == 1 ? r[1] : 0u) << 32) | r[0];
            v = __ull2double_rn(mag);
            v = ldexp(v, -(emu + e_nu[j]));
        } else {
            const int lz = __clz(r[top]);
            // 96-bit window r[top], r[top-1], r[top-2] shifted left by lz
            const uint64_t hi = (static_cast<uint64_t>(r[top]) << 32) | r[top - 1];
            uint64_t top64 = lz ? (hi << lz) | (static_cast<uint64_t>(r[top - 2]) >> (32 - lz)) : hi;
            bool sticky = lz ? (static_cast<uint32_t>(r[top - 2] << lz) != 0u) : (r[top - 2] != 0u);
            for (int t = 0; t < top - 2; ++t) sticky |= (r[t] != 0u);
            top64 |= sticky ? 1ull : 0ull;
            v = __ull2double_rn(top64);
            // value = top64 * 2^(32*(top-1) - lz)
            v = ldexp(v, 32 * (top - 1) - lz - (emu + e_nu[j]));
        }
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
