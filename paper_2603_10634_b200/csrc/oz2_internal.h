// oz2_internal.h -- shared between the host planner/launcher (oz2_api.cu) and the
// kernels.  Plain structs passed to kernels by value (they live in the constant
// parameter bank, so uniform reads are broadcasts).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace oz2 {

constexpr int kMaxModuli = 33;   // N < 34
// scaling exponent of a row / column holding NaN or Inf (R12): its entries of C are NaN
constexpr int kExpNonFinite = -2147483647 - 1;
constexpr int kMaxLimbs = 12;
constexpr int kPow2Tab = 1024;   // 2^E mod p for E in [0, 1024)
constexpr int kMaxK = 65536;     // exactness window of one FP32 accumulation
constexpr int64_t kMaxKTotal = int64_t(1) << 22;   // longer k runs in 2^16 segments (NEXT-2)
// rows of op(A) / columns of op(B): the conversion kernels put 32-row tiles in gridDim.y
constexpr int64_t kMaxRows = int64_t(65535) * 32;

// ---- GEMM (tcgen05) ------------------------------------------------------------
constexpr int BM = 128;          // rows of A per CTA tile (TMEM lanes)
constexpr int BN = 256;          // rows of B^T per CTA tile (TMEM columns per slot)
constexpr int BK = 128;          // bytes (= E4M3 elements) of K per pipeline stage
constexpr int STAGES = 4;        // CG = 1: 48 KiB per stage
constexpr int STAGES2 = 6;       // CG = 2: 32 KiB per stage per CTA
constexpr int SMEM_A_STAGE = BM * BK;   // 16 KiB
constexpr int SMEM_B_STAGE = BN * BK;   // 32 KiB
constexpr int GEMM_THREADS = 320;       // warp0 TMA, warp1 MMA, warps 2..9 epilogue
constexpr int PAD_M = 256;       // row padding of operand planes (tile multiple)
constexpr int PAD_N = 256;
constexpr int PAD_K = 128;
// Digit-plane layout: rows in blocks of kRowBlk = 128, the K extent of
// every plane cut into super-chunks of S = kSuper bytes; byte (plane x, row r, k index h) at
//   (((r / 128) KS + h / S) M + x) 128 S + (r mod 128) S + h mod S,
//   S = super_bytes(k_pad), KS = k_pad / S,
// i.e. one (row block, super-chunk) holds the M planes one after the other, each a
// contiguous 128-row x S-byte slab.  A GEMM TMA box (<= 128 rows x 128 bytes of one plane)
// stays inside one 256 KB slab (TLB locality: a per-row stride of M k_pad bytes cost 22 % of
// residue-GEMM time at k = 32768, measured), each plane keeps S contiguous bytes of K per
// row (DRAM page / L2-promotion locality: 128-byte runs cost 6 % at k = 16384), and a digit
// kernel thread stores its planes at compile-time offsets x 128 S from one address.
constexpr int kSuper = 2048;
constexpr int kRowBlk = 128;
// k_pad: a multiple of kSuper, so every call takes the specialised digit kernels (compile-time
// plane pitch); only ceil(k / 128) k-blocks are ever written or read, the rest of the last
// super-chunk is untouched address space
__host__ __device__ inline int64_t pad_k(int64_t k) {
    return (k + kSuper - 1) / kSuper * kSuper;
}
__host__ __device__ inline int64_t super_bytes(int64_t k_pad) { return k_pad < kSuper ? k_pad : kSuper; }
// byte offset of (plane x of gplanes, row r, k index h)
__host__ __device__ inline int64_t plane_offset(int64_t r, int64_t h, int x, int gplanes, int64_t k_pad) {
    const int64_t S = super_bytes(k_pad), KS = k_pad / S;
    return ((((r / kRowBlk) * KS + h / S) * gplanes + x) * kRowBlk + (r % kRowBlk)) * S + h % S;
}

// Persistent-GEMM tile order: groups of G tile-rows swept column by column (the ~148
// concurrently running tiles cover a near-square block of C and share their A and B panels
// in L2).  t -> (tile row tm, tile column tn) of a grid of m_tiles x n_tiles tiles.  Shared by
// the GEMM kernels and the tail-tile CRT (k_crt_tiles) of the hybrid schedule.
__host__ __device__ __forceinline__ void tile_coords_g(int t, int G, int m_tiles, int n_tiles, int& tm, int& tn) {
    const int group = t / (G * n_tiles);
    const int first_m = group * G;
    const int gm = G < m_tiles - first_m ? G : m_tiles - first_m;
    const int in = t - group * G * n_tiles;
    tm = first_m + in % gm;
    tn = in / gm;
}

// FP8 (kind::f8f6f4, E4M3 -> FP32) modes, and the same three on the INT8 tensor path
// (kind::i8, S8/U8 -> S32) of the INT8 Ozaki-II scheme (NEXT-3): MODE_X_I8 = MODE_X + 3
enum GemmMode : int {
    MODE_RESIDUE = 0, MODE_BOUND = 1, MODE_RAW = 2,
    MODE_RESIDUE_I8 = 3, MODE_BOUND_I8 = 4, MODE_RAW_I8 = 5
};

// moduli families (the scheme of the call)
enum Family : int { FAMILY_HYBRID_FP8 = 0, FAMILY_INT8 = 1, FAMILY_KARATSUBA_FP8 = 2 };

// ---- CRT ------------------------------------------------------------------------
struct CrtParams {
    int num_moduli;
    int p[kMaxModuli];
    uint32_t qp32[kMaxModuli];                   // round(2^32 q_l / p_l)
    uint32_t w[kMaxModuli][kMaxLimbs];           // w_l mod 2^(32L)
    uint32_t np[kMaxLimbs];                      // 2^(32L) - P
    uint32_t P[kMaxLimbs];
    uint32_t halfP[kMaxLimbs];                   // P / 2 (P is even: 1024 | P)
};

struct ModEpi {          // per modulus, residue-GEMM epilogue
    float p, pinv;
    float w16;           // smod(2^16, p): INT32 accumulators are split as hi 2^16 + lo
    float coef[3];       // square: (s, s, 1); non-square: (240, -15, 16); INT8: (1)
    int a_plane[3];      // digit-plane index of the A operand of product x
    int b_plane[3];
    int nprod;           // products (accumulator drains) of this modulus: 3, 1 (INT8) or 2
                         // (square, K-concatenated cross products)
    int a_plane2;        // >= 0: product 0 has a second part a_plane2 x b_plane2 accumulated
    int b_plane2;        // into the same TMEM accumulator (A1 B2 + A2 B1, k <= 2^15)
};

struct GemmParams {
    int m, n;                    // true sizes (store masks)
    int num_k_blocks;
    int num_kseg;                // residue mode: K segments of <= kseg_blocks k-blocks
    int kseg_blocks;             // 512 (= 2^16 / BK): FP32 exactness window per segment
    int m_tiles, n_tiles;
    int super_shift;             // log2(S / BK): k-block kb sits in super-chunk kb >> shift at
                                 // byte (kb mod 2^shift) BK (digit planes);
                                 // 30 for a plain [rows][k] matrix (raw GEMM)
    int row_blocked;             // 1: digit-plane maps {S, 128 rows, plane, super-chunk, row
                                 // block}; 0: plain maps {k, rows, 1, 1, 1}
    int num_moduli;
    int tail_head;               // residue mode: tiles [0, head) tile-major, the rest as
                                 // (tile, modulus) items (no fused CRT unless head = all tiles)
    int16_t* residues;           // [N][n][m]
    uint32_t* rmax;              // [m] float bits (bound)
    uint32_t* smax;              // [n]
    float* c32;                  // raw: [m][n]
    unsigned long long* progress;  // chip-wide product counter (progress throttle)
    // fused CRT + inverse scaling epilogue (MODE_RESIDUE, FL > 0)
    const int32_t* e_mu;
    const int32_t* e_nu;
    double alpha, beta;
    double* C;
    int64_t ldc;
    CrtParams crt;
    unsigned long long hint_a, hint_b;   // L2 cache policies of the operand TMA loads
    int sync_lead;               // 0 = off; else max chunks ahead of the chip-wide average
    int sync_chunk;              // k-blocks per throttle chunk (0 = one chunk per product)
    int prods_per_tile;          // residue mode: sum of mod[l].nprod (accumulator drains per tile)
    int max_units;               // host only: cap on persistent units (0 = all)
    unsigned epi_sleep_ns;       // residue mode: epilogue poll interval while an accumulator fills
    ModEpi mod[kMaxModuli];
};

// ---- residue / digit split ------------------------------------------------------
constexpr int kNumSquares = 6;   // square moduli lead the hybrid list (33^2 ... 23^2)

struct ModDig {
    double p_d, pinv_d;
    float p_f, pinv_f, s_f, inv_s_f;
    float hp_f;                  // (p even ? 1/2 : 0) / p: offset of the symmetric rounding
    float h_f;                   // p even ? 1/2 : 0
    float w8[8];                 // smod(2^(8i), p) as floats: byte-chunk weights
    int square;
    int plane0;                  // first digit plane of this modulus
    double q2_d, q2inv_d;        // paired residues (k_digits, |X'| < lim1): Q = p_l p_(l+1)
                                 // for even l < N-1 (else Q = p_l), and RN(1/Q)
};

struct DigitParams {
    int num_moduli;
    int num_planes;
    int int8;                    // 1: INT8 scheme (one S8 residue plane per modulus)
    int num_squares;             // FP8: leading square moduli (hybrid min(N, 6), Karatsuba 0)
    int even_index;              // index of the (single, by coprimality) even modulus, or -1
    // reduction-depth limits on |X'|: the 1.5 2^52 rounding trick needs |q| <= 2^51, so
    // one FP64 step serves |X'| < 2^50 p_min and the p 2^36 pre-reduction |X'| < 2^86 p_min
    double lim1, lim2;
    const uint16_t* pow2tab;     // [N][kPow2Tab]
    ModDig mod[kMaxModuli];
};

// ---- exponents ------------------------------------------------------------------
struct ExpParams {
    float p_prime, delta, f_k;
};

// fast mode: H = RD64((P-1)/2) = h 2^th, h < 2^53 (reading R15)
struct FastExpParams {
    unsigned long long h;
    int th;
};

// launchers (defined in the .cu files)
cudaError_t launch_rowmax(const double* X, int64_t rows, int64_t k, int64_t ld, bool kmajor,
                          unsigned long long* maxbits, cudaStream_t st);
cudaError_t launch_cast(const double* X, int64_t rows, int64_t k, int64_t ld, bool kmajor,
                        const unsigned long long* maxbits, int32_t* eprime, uint8_t* xbar, int gplanes,
                        int64_t rows_pad, int64_t k_pad, int32_t* status,
                        unsigned long long* sumsq, bool i8, cudaStream_t st);
// one-read prescale (accurate mode): chunk-local casts + rescale to the row exponent
cudaError_t launch_cast_local(const double* X, int64_t rows, int64_t k, int64_t ld, bool kmajor,
                              unsigned long long* maxbits, int16_t* eloc, uint8_t* xbar, int gplanes,
                              int64_t rows_pad, int64_t k_pad, bool i8, cudaStream_t st);
cudaError_t launch_rescale(int64_t rows, int64_t k, const unsigned long long* maxbits, const int16_t* eloc,
                           int32_t* eprime, int32_t* status, uint8_t* xbar, int gplanes, int64_t k_pad, bool i8,
                           cudaStream_t st);
cudaError_t launch_exps_fast(const unsigned long long* maxbits, const int32_t* eprime,
                             const unsigned long long* sumsq, const uint32_t* u32, int64_t count,
                             FastExpParams fp, int ushift, int32_t* e_out, cudaStream_t st);
cudaError_t launch_exps(const unsigned long long* maxbits, const int32_t* eprime,
                        const uint32_t* rsmax, int64_t count, ExpParams ep, int32_t* e_out,
                        cudaStream_t st);
// maxbits: step 1's row maxima of |X| (selects the one-FMA fast path per row), or nullptr
cudaError_t launch_digits(const double* X, int64_t rows, int64_t k, int64_t ld, bool kmajor,
                          const int32_t* e, const unsigned long long* maxbits, const DigitParams& dp, uint8_t* planes,
                          int64_t rows_pad, int64_t k_pad, cudaStream_t st);
// plane x of the digit-plane layout (gplanes planes per super-chunk group) -> dst [rows][k]
cudaError_t launch_unpack_plane(uint8_t* dst, const uint8_t* src, int gplanes, int x, int64_t rows, int64_t k,
                                int64_t k_pad, cudaStream_t st);
cudaError_t launch_gemm(int mode, int cg, int fused_limbs, const CUtensorMap& ta, const CUtensorMap& tb,
                        const GemmParams& gp, int num_sms, cudaStream_t st, int tile_n = 256);
cudaError_t launch_res_symmetric(int16_t* out, const int16_t* in, int64_t per, const CrtParams& cp,
                                 cudaStream_t st);
cudaError_t launch_crt(int limbs, const int16_t* res, int64_t m, int64_t n, const CrtParams& cp,
                       const int32_t* e_mu, const int32_t* e_nu, double alpha, double beta,
                       double* C, int64_t ldc, bool generic, cudaStream_t st);
cudaError_t launch_scale(double* C, int64_t m, int64_t n, int64_t ldc, double beta, cudaStream_t st);
// CRT + inverse scaling of the tiles [t0, t0 + count) of the residue GEMM's tile order (the
// split tail of the hybrid schedule when the CRT of the other tiles is fused): tile t covers
// rows tm tile_rows .. and columns tn tile_cols .. (tile_coords_g with G)
cudaError_t launch_crt_tiles(int limbs, const int16_t* res, int64_t m, int64_t n, const CrtParams& cp,
                             const int32_t* e_mu, const int32_t* e_nu, double alpha, double beta, double* C,
                             int64_t ldc, int t0, int count, int G, int m_tiles, int n_tiles, int tile_rows,
                             int tile_cols, cudaStream_t st);

}  // namespace oz2
