// crt_kernel.cu -- standalone Chinese-remainder reconstruction + inverse scaling
// (eq. CRT_finalreduction, eq. inversescaling); the arithmetic is in
// crt_common.cuh (shared with the fused residue-GEMM epilogue).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "oz2_internal.h"
#include "crt_common.cuh"

namespace oz2 {

template <int L>
__global__ void __launch_bounds__(256) k_crt(const int16_t* __restrict__ res, int64_t m, int64_t n,
                                             const __grid_constant__ CrtParams cp,
                                             const int32_t* __restrict__ e_mu,
                                             const int32_t* __restrict__ e_nu, double alpha,
                                             double beta, double* __restrict__ C, int64_t ldc) {
    __shared__ CrtShared s;
    crt_stage_constants(&s, cp, threadIdx.x, blockDim.x);
    __syncthreads();
    const int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    if (i >= m) return;
    const int emu = e_mu[i];
    const int64_t lstride = n * m;
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
        const int enu = e_nu[j];
        const double v = exps_finite(emu, enu) ? crt_element<L>(res + j * m + i, lstride, &s, cp, emu + enu, false)
                                               : __longlong_as_double(0x7FF8000000000000ll);
        store_alpha_beta(C + i + j * ldc, v, alpha, beta);
    }
}

// Specialised for the common (limbs, moduli) pairs: two consecutive rows per thread (one
// 32-bit load per modulus), all NM residue loads issued before the arithmetic, and the
// CRT weights read straight from the kernel-parameter constant bank (fully unrolled).
template <int L, int NM>
__global__ void __launch_bounds__(256, 4) k_crt_n(const int16_t* __restrict__ res, int64_t m, int64_t n,
                                               const __grid_constant__ CrtParams cp,
                                               const int32_t* __restrict__ e_mu,
                                               const int32_t* __restrict__ e_nu, double alpha,
                                               double beta, double* __restrict__ C, int64_t ldc) {
    const int64_t i = 2 * (static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x);   // m is even
    if (i >= m) return;
    const int emu0 = e_mu[i], emu1 = e_mu[i + 1];
    const int64_t lstride = n * m;
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
        const unsigned int* rp = reinterpret_cast<const unsigned int*>(res + j * m + i);
        const int64_t ls2 = lstride / 2;                 // in 32-bit words (lstride is even)
        uint32_t rr[NM];
#pragma unroll
        for (int l = 0; l < NM; ++l) {
            rr[l] = __ldcs(rp);
            rp += ls2;
        }
        const int enu = e_nu[j];
        // both rows accumulate in one pass over the moduli, so each CRT weight (a uniform
        // constant) is fetched once per modulus for the two elements
        uint64_t acc0[L], acc1[L];
#pragma unroll
        for (int t = 0; t < L; ++t) { acc0[t] = 0; acc1[t] = 0; }
        uint64_t tacc0 = 0x80000000ull, tacc1 = 0x80000000ull;
#pragma unroll
        for (int l = 0; l < NM; ++l) {
            const uint32_t u0 = rr[l] & 0xFFFFu, u1 = rr[l] >> 16;         // u_l in [0, p_l)
            const uint32_t qp = cp.qp32[l];
            tacc0 += static_cast<uint64_t>(u0) * qp;
            tacc1 += static_cast<uint64_t>(u1) * qp;
#pragma unroll
            for (int t = 0; t < L; ++t) {
                const uint32_t wv = cp.w[l][t];
                acc0[t] += static_cast<uint64_t>(u0) * wv;
                acc1[t] += static_cast<uint64_t>(u1) * wv;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int emu = h ? emu1 : emu0;
            const double v = !exps_finite(emu, enu) ? __longlong_as_double(0x7FF8000000000000ll)
                           : h ? crt_finish<L>(acc1, tacc1, cp, emu + enu) : crt_finish<L>(acc0, tacc0, cp, emu + enu);
            store_alpha_beta(C + i + h + j * ldc, v, alpha, beta);
        }
    }
}

// CRT of whole tiles of the residue GEMM's tile order (the split tail of the hybrid schedule;
// the other tiles' CRT is fused into the GEMM epilogue).  Block (x, y): tile t0 + x, thread =
// one row of the tile, columns y, y + gridDim.y, ... of the tile.
template <int L>
__global__ void __launch_bounds__(256) k_crt_tiles(const int16_t* __restrict__ res, int64_t m, int64_t n,
                                                   const __grid_constant__ CrtParams cp,
                                                   const int32_t* __restrict__ e_mu,
                                                   const int32_t* __restrict__ e_nu, double alpha, double beta,
                                                   double* __restrict__ C, int64_t ldc, int t0, int G, int m_tiles,
                                                   int n_tiles, int tile_rows, int tile_cols) {
    __shared__ CrtShared s;
    crt_stage_constants(&s, cp, threadIdx.x, blockDim.x);
    __syncthreads();
    int tm, tn;
    tile_coords_g(t0 + static_cast<int>(blockIdx.x), G, m_tiles, n_tiles, tm, tn);
    const int64_t lstride = n * m;
    for (int rr = threadIdx.x; rr < tile_rows; rr += blockDim.x) {
        const int64_t i = static_cast<int64_t>(tm) * tile_rows + rr;
        if (i >= m) break;
        const int emu = e_mu[i];
        for (int jj = blockIdx.y; jj < tile_cols; jj += gridDim.y) {
            const int64_t j = static_cast<int64_t>(tn) * tile_cols + jj;
            if (j >= n) break;
            const int enu = e_nu[j];
            const double v = exps_finite(emu, enu) ? crt_element<L>(res + j * m + i, lstride, &s, cp, emu + enu, false)
                                                   : __longlong_as_double(0x7FF8000000000000ll);
            store_alpha_beta(C + i + j * ldc, v, alpha, beta);
        }
    }
}

cudaError_t launch_crt_tiles(int limbs, const int16_t* res, int64_t m, int64_t n, const CrtParams& cp,
                             const int32_t* e_mu, const int32_t* e_nu, double alpha, double beta, double* C,
                             int64_t ldc, int t0, int count, int G, int m_tiles, int n_tiles, int tile_rows,
                             int tile_cols, cudaStream_t st) {
    if (count <= 0 || m == 0 || n == 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>(count), 32u);
#define OZ2_CRTT_CASE(LL)                                                                                     \
    case LL:                                                                                                  \
        k_crt_tiles<LL><<<grid, 256, 0, st>>>(res, m, n, cp, e_mu, e_nu, alpha, beta, C, ldc, t0, G, m_tiles, \
                                              n_tiles, tile_rows, tile_cols);                                 \
        break;
    switch (limbs) {
        OZ2_CRTT_CASE(4)
        OZ2_CRTT_CASE(5)
        OZ2_CRTT_CASE(6)
        default: return cudaErrorInvalidValue;    // the fused CRT (hence this tail) needs <= 6 limbs
    }
#undef OZ2_CRTT_CASE
    return cudaGetLastError();
}

// debug output: the stored u_l in [0, p_l) back to the symmetric range of C'_l (R2)
__global__ void k_res_symmetric(int16_t* __restrict__ out, const int16_t* __restrict__ in, int64_t per,
                                const __grid_constant__ CrtParams cp) {
    const int l = blockIdx.y;
    const int p = cp.p[l];
    const int half = (p + 1) / 2;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < per;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int u = static_cast<uint16_t>(in[l * per + e]);
        out[l * per + e] = static_cast<int16_t>(u >= half ? u - p : u);
    }
}

cudaError_t launch_res_symmetric(int16_t* out, const int16_t* in, int64_t per, const CrtParams& cp,
                                 cudaStream_t st) {
    if (per == 0) return cudaSuccess;
    const int64_t bx = (per + 255) / 256;
    dim3 grid(static_cast<unsigned>(bx < 4096 ? bx : 4096), static_cast<unsigned>(cp.num_moduli));
    k_res_symmetric<<<grid, 256, 0, st>>>(out, in, per, cp);
    return cudaGetLastError();
}

cudaError_t launch_crt(int limbs, const int16_t* res, int64_t m, int64_t n, const CrtParams& cp,
                       const int32_t* e_mu, const int32_t* e_nu, double alpha, double beta,
                       double* C, int64_t ldc, bool generic, cudaStream_t st) {
    if (m == 0 || n == 0) return cudaSuccess;
    // ~2048 blocks in total, each looping over many columns (amortises the staging of
    // the CRT constants in shared memory)
    if (m % 2 == 0 && !generic) {          // generic: OZ2_TUNE_CRT_GENERIC (A/B reference)
        const int64_t gx2 = (m / 2 + 255) / 256;
        int64_t gy2 = 2048 / gx2;
        gy2 = gy2 < 1 ? 1 : (gy2 > n ? n : gy2);
        dim3 grid2(static_cast<unsigned>(gx2), static_cast<unsigned>(gy2 < 65535 ? gy2 : 65535));
#define OZ2_CRTN(LL, NN)                                                                            \
        if (limbs == LL && cp.num_moduli == NN) {                                                   \
            k_crt_n<LL, NN><<<grid2, 256, 0, st>>>(res, m, n, cp, e_mu, e_nu, alpha, beta, C, ldc); \
            return cudaGetLastError();                                                              \
        }
        OZ2_CRTN(4, 12) OZ2_CRTN(4, 13) OZ2_CRTN(4, 14) OZ2_CRTN(4, 15) OZ2_CRTN(5, 15)
        OZ2_CRTN(5, 16) OZ2_CRTN(4, 16) OZ2_CRTN(5, 17) OZ2_CRTN(5, 18) OZ2_CRTN(6, 20)
#undef OZ2_CRTN
    }
    const int64_t gx = (m + 255) / 256;
    int64_t gy = 2048 / gx;
    gy = gy < 1 ? 1 : (gy > n ? n : gy);
    dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy < 65535 ? gy : 65535));
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
