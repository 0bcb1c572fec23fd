// gemm_kernel.cu -- the FP8 (E4M3 x E4M3 -> FP32) GEMMs of the FP8 Ozaki-II scheme on
// 5th-generation tensor cores (tcgen05.mma kind::f8f6f4), one persistent CTA per SM.
//
// Roles (320 threads):
//   warp 0      TMA producer: A tile 128 x 128 B and B tile 256 x 128 B per stage,
//               128-byte swizzle, 4-stage mbarrier ring
//   warp 1      TMEM allocator + single-thread MMA issuer: 4 x (M=128, N=256, K=32)
//               MMAs per stage into one of two 256-column FP32 accumulators in TMEM
//   warps 2..9  epilogue: tcgen05.ld 32 lanes x 32 columns, each warp owns a TMEM lane
//               quadrant (warp % 4) and one 128-column half of the tile
//
// Modes:
//   MODE_RESIDUE  for every tile and every modulus l the three exact products of
//                 P:292-299 (square p = s^2: A1 B2, A2 B1, A2 B2 with weights s, s, 1)
//                 or eq. C'-Karatsuba P:241-246 (non-square: A^x B^x, x = 1..3 with
//                 weights 256-16, 1-16, 16) run back to back; the epilogue reduces
//                 each FP32 accumulator mod p (exact: entries are integers <= 2^24,
//                 eq. error-free-FP8-matmult) and accumulates the weighted partial in
//                 registers; after the third product it writes C'_l = mod(.., p) as
//                 int16 [l][j][i].  The FP32 products never leave TMEM.
//   MODE_BOUND    C-bar' = A-bar B-bar; the epilogue keeps only the row and
//                 column maxima (atomicMax on non-negative float bits).
//   MODE_RAW      diagnostic: writes the FP32 accumulator.
#include <cstdint>
#include <cuda_runtime.h>
#include "oz2_internal.h"
#include "oz2_ptx.cuh"
#include <cuda_fp16.h>

namespace oz2 {

__device__ __forceinline__ void tile_coords(int t, int m_tiles, int n_tiles, int& tm, int& tn) {
    // groups of 16 tile-rows swept column by column: concurrently running CTAs share
    // A and B panels in L2
    constexpr int G = 16;
    const int group = t / (G * n_tiles);
    const int first_m = group * G;
    const int gm = min(G, m_tiles - first_m);
    const int in = t - group * G * n_tiles;
    tm = first_m + in % gm;
    tn = in / gm;
}

template <int MODE>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const __grid_constant__ GemmParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * SMEM_A_STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * SMEM_B_STAGE);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = warp_id_uniform();
    const uint32_t lane = lane_id();

    if (warp == 0) {
        if (elect_one()) {
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 1);
            }
            for (int s = 0; s < 2; ++s) {
                mbar_init(&tfull[s], 1);
                mbar_init(&tempty[s], 8);
            }
            fence_mbar_init();
        }
        __syncwarp();
    } else if (warp == 1) {
        tmem_alloc(tmem_slot, 512);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int num_tiles = P.m_tiles * P.n_tiles;
    const int prods = (MODE == MODE_RESIDUE) ? 3 * P.num_moduli : 1;
    const int nkb = P.num_k_blocks;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (elect_one()) {
            uint32_t stage = 0, phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int tm, tn;
                tile_coords(tile, P.m_tiles, P.n_tiles, tm, tn);
                for (int pr = 0; pr < prods; ++pr) {
                    int a_row = tm * BM, b_row = tn * BN;
                    if (MODE == MODE_RESIDUE) {
                        const int l = pr / 3, x = pr - 3 * (pr / 3);
                        a_row += P.mod[l].a_plane[x] * P.rows_per_plane_a;
                        b_row += P.mod[l].b_plane[x] * P.rows_per_plane_b;
                    }
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        mbar_arrive_expect_tx(&full[stage], SMEM_A_STAGE + SMEM_B_STAGE);
                        tma_load_2d(&tmA, &full[stage], sA + stage * SMEM_A_STAGE, kb * BK, a_row, kEvictNormal);
                        tma_load_2d(&tmB, &full[stage], sB + stage * SMEM_B_STAGE, kb * BK, b_row, kEvictNormal);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (elect_one()) {
            constexpr uint32_t idesc = make_idesc_e4m3_f32(BM, BN);
            uint32_t stage = 0, phase = 0, g = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                for (int pr = 0; pr < prods; ++pr, ++g) {
                    const uint32_t slot = g & 1u, use = g >> 1;
                    mbar_wait(&tempty[slot], (use & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + slot * BN;
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint64_t a0 = make_desc_k128_sw128(smem_u32(sA + stage * SMEM_A_STAGE));
                        const uint64_t b0 = make_desc_k128_sw128(smem_u32(sB + stage * SMEM_B_STAGE));
#pragma unroll
                        for (int kk = 0; kk < BK / 32; ++kk) {
                            // advance 32 bytes of K inside the 128-byte swizzle atom
                            mma_f8f6f4(d_tmem, a0 + 2 * kk, b0 + 2 * kk, idesc, (kb | kk) != 0);
                        }
                        mma_commit(&empty[stage]);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    mma_commit(&tfull[slot]);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const uint32_t quad = warp & 3u;           // TMEM lane quadrant this warp may access
        const uint32_t half = (warp - 2u) >> 2;    // 128-column half of the 256-column tile
        const uint32_t row_in_tile = quad * 32u + lane;
        uint32_t g = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            int tm, tn;
            tile_coords(tile, P.m_tiles, P.n_tiles, tm, tn);
            const int64_t row = static_cast<int64_t>(tm) * BM + row_in_tile;
            const int64_t col0 = static_cast<int64_t>(tn) * BN + half * 128u;
            if (MODE == MODE_RESIDUE) {
                for (int l = 0; l < P.num_moduli; ++l) {
                    const float p = P.mod[l].p, pinv = P.mod[l].pinv;
                    // running partial sum_x coef_x r_x, reduced mod p after every product
                    // (|.| <= p/2 + 1 <= 546), held exactly in binary16 pairs
                    __half2 part[64];
                    int16_t* out = P.residues + (static_cast<int64_t>(l) * P.n + col0) * P.m + row;
                    const bool row_ok = row < P.m;
#pragma unroll
                    for (int x = 0; x < 3; ++x, ++g) {
                        const float coef = P.mod[l].coef[x];
                        const uint32_t slot = g & 1u, use = g >> 1;
                        mbar_wait(&tfull[slot], use & 1u);
                        tc_fence_after();
                        const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + slot * BN + half * 128u;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            uint32_t v[32];
                            tmem_ld_32x32b_x32(taddr + c * 32, v);
                            tmem_ld_wait();
#pragma unroll
                            for (int j = 0; j < 32; j += 2) {
                                float acc[2];
#pragma unroll
                                for (int u = 0; u < 2; ++u) {
                                    const float f = __uint_as_float(v[j + u]);       // exact integer, |f| <= 2^24
                                    const float r = fmaf(-rintf(f * pinv), p, f);    // f mod p, |r| <= p/2 + 1
                                    acc[u] = r;
                                }
                                const int idx = (c * 32 + j) >> 1;
                                if (x == 0) {
                                    acc[0] *= coef;
                                    acc[1] *= coef;
                                } else {
                                    const float2 pv = __half22float2(part[idx]);
                                    acc[0] = fmaf(coef, acc[0], pv.x);
                                    acc[1] = fmaf(coef, acc[1], pv.y);
                                }
#pragma unroll
                                for (int u = 0; u < 2; ++u) acc[u] = fmaf(-rintf(acc[u] * pinv), p, acc[u]);
                                if (x < 2) {
                                    part[idx] = __floats2half2_rn(acc[0], acc[1]);  // exact (|acc| <= 546)
                                } else {
                                    // C'_l = mod(sum_x coef_x r_x, p), symmetric range (R2)
#pragma unroll
                                    for (int u = 0; u < 2; ++u) {
                                        float r = acc[u];
                                        if (2.0f * r >= p) r -= p;
                                        else if (2.0f * r < -p) r += p;
                                        const int jj = c * 32 + j + u;
                                        if (row_ok && col0 + jj < P.n)
                                            out[static_cast<int64_t>(jj) * P.m] = static_cast<int16_t>(r);
                                    }
                                }
                            }
                        }
                        // accumulator slot drained: hand it back to the MMA warp
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[slot]);
                    }
                }
            } else {
                const uint32_t slot = g & 1u, use = g >> 1;
                mbar_wait(&tfull[slot], use & 1u);
                tc_fence_after();
                const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + slot * BN + half * 128u;
                float rowmax = 0.0f;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(taddr + c * 32, v);
                    tmem_ld_wait();
                    if (MODE == MODE_BOUND) {
                        uint32_t mycol = 0;
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            rowmax = fmaxf(rowmax, __uint_as_float(v[j]));
                            const uint32_t cm = __reduce_max_sync(0xffffffffu, v[j]);
                            if (lane == static_cast<uint32_t>(j)) mycol = cm;
                        }
                        const int64_t col = col0 + c * 32 + lane;
                        if (col < P.n && mycol) atomicMax(P.smax + col, mycol);
                    } else if (row < P.m) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int64_t col = col0 + c * 32 + j;
                            if (col < P.n) P.c32[row * P.n + col] = __uint_as_float(v[j]);
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[slot]);
                ++g;
                if (MODE == MODE_BOUND && row < P.m && rowmax > 0.0f)
                    atomicMax(P.rmax + row, __float_as_uint(rowmax));
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

static bool g_attr_set[3] = {false, false, false};

cudaError_t launch_gemm(int mode, const CUtensorMap& ta, const CUtensorMap& tb,
                        const GemmParams& gp, int num_sms, cudaStream_t st) {
    const int num_tiles = gp.m_tiles * gp.n_tiles;
    if (num_tiles == 0) return cudaSuccess;
    const int grid = num_tiles < num_sms ? num_tiles : num_sms;
    cudaError_t err = cudaSuccess;
    switch (mode) {
        case MODE_RESIDUE:
            if (!g_attr_set[0]) {
                err = cudaFuncSetAttribute(gemm_kernel<MODE_RESIDUE>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
                if (err != cudaSuccess) return err;
                g_attr_set[0] = true;
            }
            gemm_kernel<MODE_RESIDUE><<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(ta, tb, gp);
            break;
        case MODE_BOUND:
            if (!g_attr_set[1]) {
                err = cudaFuncSetAttribute(gemm_kernel<MODE_BOUND>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
                if (err != cudaSuccess) return err;
                g_attr_set[1] = true;
            }
            gemm_kernel<MODE_BOUND><<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(ta, tb, gp);
            break;
        default:
            if (!g_attr_set[2]) {
                err = cudaFuncSetAttribute(gemm_kernel<MODE_RAW>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
                if (err != cudaSuccess) return err;
                g_attr_set[2] = true;
            }
            gemm_kernel<MODE_RAW><<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(ta, tb, gp);
            break;
    }
    return cudaGetLastError();
}

}  // namespace oz2
