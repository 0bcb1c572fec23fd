// crt_kernel.cu -- standalone Chinese-remainder reconstruction + inverse scaling
// (eq. CRT_finalreduction, eq. inversescaling); the arithmetic is in
// crt_common.cuh (shared with the fused residue-GEMM epilogue).
#include <cstdint>
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
        const double v = crt_element<L>(res + j * m + i, lstride, &s, cp, emu + e_nu[j], false);
        store_alpha_beta(C + i + j * ldc, v, alpha, beta);
    }
}

cudaError_t launch_crt(int limbs, const int16_t* res, int64_t m, int64_t n, const CrtParams& cp,
                       const int32_t* e_mu, const int32_t* e_nu, double alpha, double beta,
                       double* C, int64_t ldc, cudaStream_t st) {
    if (m == 0 || n == 0) return cudaSuccess;
    // ~2048 blocks in total, each looping over many columns (amortises the staging of
    // the CRT constants in shared memory)
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
