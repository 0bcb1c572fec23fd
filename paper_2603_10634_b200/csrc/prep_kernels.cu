// prep_kernels.cu -- the HBM-bound conversion kernels of the FP8 Ozaki-II pipeline.
//
//   k_rowmax  max_h |x_rh| per operand row (for mu', nu'; eq. def:mu'nu')
//   k_cast    e'_r = 7 - floor(log2 max) and X-bar = RU_fp8(|x| 2^e')
//   k_exps    log2 mu = log2 mu' + int(P' + delta log2 RU(f_k R))      (eq. mu-computation)
//   k_digits  X' = trunc(2^e x), residues mod p_l, FP8 digit split
//
// An operand is seen as `rows` rows of length k (A: rows = i; B: rows = j of B^T).
// Element (r, h) lives at X[r + h*ld] (MN-major: A with transa='N', B with 'T') or
// X[h + r*ld] (K-major: A 'T', B 'N').  Outputs are K-major byte planes in the row-blocked
// super-chunk layout (plane_offset in oz2_internal.h): per 128-row block
// and S-wide K super-chunk, the M planes are consecutive 128-row x S-byte slabs, so (S =
// kSuper) a thread's stores to its planes differ by compile-time multiples of 128 S bytes.
// Zero in the padding.
#include <cstdint>
#include <cuda_runtime.h>
#include "oz2_internal.h"
#include "oz2_ptx.cuh"

namespace oz2 {

// ---------------------------------------------------------------------------------
// row maxima of |x| as binary64 bit patterns (non-negative doubles order like their
// bits; NaN/Inf patterns sort above every finite value and are flagged in k_cast)

template <bool KMAJOR>
__global__ void __launch_bounds__(256) k_rowmax(const double* __restrict__ X, int64_t rows,
                                                int64_t k, int64_t ld,
                                                unsigned long long* __restrict__ maxbits) {
    if (!KMAJOR) {
        // thread per row, block strip of k; coalesced across the rows
        const int64_t r = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
        const int64_t h0 = static_cast<int64_t>(blockIdx.y) * 512;
        const int64_t h1 = min(k, h0 + 512);
        if (r >= rows) return;
        unsigned long long mx = 0;
        const double* p = X + r + h0 * ld;
#pragma unroll 8
        for (int64_t h = h0; h < h1; ++h, p += ld) {
            const unsigned long long b = __double_as_longlong(fabs(__ldg(p)));
            mx = b > mx ? b : mx;
        }
        if (mx) atomicMax(maxbits + r, mx);
    } else {
        // warp per row, lanes stride along k
        const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
        if (r >= rows) return;
        const double* p = X + r * ld;
        unsigned long long mx = 0;
        int64_t h = threadIdx.x & 31;
        for (; h + 96 < k; h += 128) {
            const double a0 = __ldg(p + h), a1 = __ldg(p + h + 32), a2 = __ldg(p + h + 64),
                         a3 = __ldg(p + h + 96);
            unsigned long long b0 = __double_as_longlong(fabs(a0)), b1 = __double_as_longlong(fabs(a1));
            unsigned long long b2 = __double_as_longlong(fabs(a2)), b3 = __double_as_longlong(fabs(a3));
            b0 = b0 > b1 ? b0 : b1;
            b2 = b2 > b3 ? b2 : b3;
            b0 = b0 > b2 ? b0 : b2;
            mx = mx > b0 ? mx : b0;
        }
        for (; h < k; h += 32) {
            const unsigned long long b = __double_as_longlong(fabs(__ldg(p + h)));
            mx = mx > b ? mx : b;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long v = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = mx > v ? mx : v;
        }
        if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxbits + r, mx);
    }
}

// floor(log2 x) of a positive finite binary64 given as bits
__device__ __forceinline__ int ilog2_bits(unsigned long long b) {
    const int ef = static_cast<int>(b >> 52);
    if (ef > 0) return ef - 1023;
    const unsigned long long mant = b & 0xFFFFFFFFFFFFFull;
    return (63 - __clzll(static_cast<long long>(mant))) - 1074;
}

template <bool I8 = false>
__device__ __forceinline__ int eprime_of(unsigned long long mb) {
    // log2 mu' = 7 - floor(log2 max|x|) (eq. def:mu'nu'); INT8 scheme: 6 - floor(...) so
    // that ceil(|x| mu') <= 128 (R16); zero row -> 0 (reading R3)
    if (mb == 0ull || mb >= 0x7FF0000000000000ull) return 0;
    return (I8 ? 6 : 7) - ilog2_bits(mb);
}

// ---------------------------------------------------------------------------------
// Tile loader shared by k_cast and k_digits: a 32-row x 128-h tile of doubles in
// shared memory (zero outside [0,rows) x [0,k)), loaded coalesced for both layouts.

constexpr int TR = 32;     // rows per tile
constexpr int TH = 128;    // k per tile
constexpr int TP = TH + 1; // padded shared row (doubles)

template <bool KMAJOR>
__device__ __forceinline__ void load_tile(const double* __restrict__ X, int64_t rows, int64_t k,
                                          int64_t ld, int64_t r0, int64_t h0, double* tile) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (!KMAJOR) {
        // each warp reads 32 consecutive rows for 16 values of h (256 B per request)
#pragma unroll 4
        for (int j = 0; j < TH / 8; ++j) {
            const int hh = w * (TH / 8) + j;
            const int64_t r = r0 + lane, h = h0 + hh;
            double v = 0.0;
            if (r < rows && h < k) v = __ldg(X + r + h * ld);
            tile[lane * TP + hh] = v;
        }
    } else {
        // each warp reads 4 rows, 128 consecutive h per row (1 KiB per row)
#pragma unroll
        for (int j = 0; j < TR / 8; ++j) {
            const int rr = w * (TR / 8) + j;
            const int64_t r = r0 + rr;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int hh = q * 32 + lane;
                const int64_t h = h0 + hh;
                double v = 0.0;
                if (r < rows && h < k) v = __ldg(X + h + r * ld);
                tile[rr * TP + hh] = v;
            }
        }
    }
}

// byte offset of (row r, 128-byte chunk c) of plane 0 in the layout with `gplanes` planes
// per group; S = kSuper (kCps chunks per super-chunk) or S = k_pad (one super-chunk)
constexpr uint32_t kCps = kSuper / TH;
__device__ __forceinline__ int64_t chunk_offset(int64_t r, uint32_t c, int gplanes, int64_t k_pad) {
    const int64_t rb = r >> 7, ri = r & (kRowBlk - 1);
    if (k_pad >= kSuper)
        return ((rb * (k_pad / kSuper) + c / kCps) * gplanes * kRowBlk + ri) * kSuper + (c % kCps) * TH;
    return (rb * gplanes * kRowBlk + ri) * k_pad + c * TH;
}

// the same for the digit planes (num_planes per group), S = kSuper known at compile time
template <bool SUP>
__device__ __forceinline__ int64_t chunk_offset_planes(int64_t r, uint32_t c, int planes, int64_t k_pad) {
    const int64_t rb = r >> 7, ri = r & (kRowBlk - 1);
    if (SUP) return ((rb * (k_pad / kSuper) + c / kCps) * planes * kRowBlk + ri) * kSuper + (c % kCps) * TH;
    return (rb * planes * kRowBlk + ri) * k_pad + c * TH;
}

__device__ __forceinline__ double pow2d(int e) {          // 2^e, |e| <= 1022
    return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
}

// ---------------------------------------------------------------------------------
// k_cast: e' and X-bar = RU_fp8(|x| 2^e')
// FAST (fast mode, reading R15): X-bar is not stored; instead S_r = sum_h xbar_rh^2 is
// accumulated exactly as an integer in units of 2^-18 (E4M3 squares are multiples of
// 2^-18 and <= 2^16, so S_r < 2^56 for k <= 2^22 and the sum is order-independent).

__device__ __forceinline__ unsigned long long fp8_sq_units(uint32_t c) {   // code^2 / 2^-18
    const uint32_t E = (c >> 3) & 15u, mt = c & 7u;
    return E ? static_cast<unsigned long long>((8u + mt) * (8u + mt)) << (2 * E - 2)
             : static_cast<unsigned long long>(mt * mt);
}

// I8 (INT8 scheme, R16): X-bar = ceil(|x| 2^e') in [0, 128] as U8 (exact upper bounds),
// squares accumulated in units of 1.
//
// No shared-memory staging (round 2, session 4): a lane converts kCastH = 16 consecutive k of a row.
//   MN-major (X[r + h ld]): lane = row, so each of the lane's 16 loads is one coalesced 256-byte
//     run per warp; warp w of a block takes k in [h0 + 16 w, h0 + 16 w + 16): block = 32 rows x
//     128 k (one 128-byte chunk of the layout), grid (rows_pad / 32, ceil(k / 128)).
//   K-major (X[h + r ld]): warp = row, lane = 8 pairs of consecutive k 64 apart (eight coalesced
//     16-byte loads when X is 16-byte aligned and ld even): block = 8 rows x 512 k, grid
//     (rows_pad / 8, ceil(k / 512)).
// The E4M3 round-up of the common element is four integer instructions on the high word of x
// (cast_code); zeros, subnormal-range results and NaN / Inf rows take a warp-divergent slow
// path.  Padding rows / k get zero codes.
constexpr int kCastH = 16;

struct CastRow {
    uint32_t thr;        // |hi(x)| >= thr: the common path is exact (x normal, |x| 2^e >= 2^-6)
    uint32_t add;        // ((e - 1016) << 20) + 0x1FFFF
    int e;
    bool bad;            // NaN / Inf row (R12): zero bounds, it cannot disturb other exponents
};

template <bool I8>
__device__ __forceinline__ CastRow cast_row(unsigned long long mb) {
    CastRow cr;
    cr.e = eprime_of<I8>(mb);
    cr.bad = mb >= 0x7FF0000000000000ull;
    // y = |x| 2^e has binary64 exponent field ey = (hx >> 20) + e; the E4M3 normal range is
    // y >= 2^-6, i.e. ey >= 1017, and x itself must be normal: hx >= max(1017 - e, 1) << 20
    const int lo = 1017 - cr.e;
    cr.thr = cr.bad ? 0xFFFFFFFFu : static_cast<uint32_t>(lo > 1 ? lo : 1) << 20;
    cr.add = static_cast<uint32_t>((cr.e - 1016) * (1 << 20) + 0x1FFFF);
    return cr;
}

// RU_e4m3(|x| 2^e) as a code for a common element (|hi(x)| >= thr): hy = hx + (e << 20) is the
// high word of y; its top 3 significand bits rounded up (sticky = the other 49 bits, via +0x1FFFF
// and min(lx, 1)) are (hy >> 17) - (1016 << 3) = (E + 7) 8 + M3, the code (R4).
__device__ __forceinline__ uint32_t cast_code(uint32_t hx, uint32_t lx, uint32_t add) {
    return (hx + add + min(lx, 1u)) >> 17;
}

template <bool I8>
__device__ __forceinline__ uint32_t cast_code_slow(double x, const CastRow& cr) {
    if (x == 0.0 || cr.bad) return 0u;
    const double s1 = pow2d(cr.e >> 1), s2 = pow2d(cr.e - (cr.e >> 1));   // 2^e in two exact steps
    if (I8) return static_cast<uint32_t>(ceil((fabs(x) * s1) * s2));     // exact: <= 2^7 scaled
    const uint32_t c = fp8_ru_code((fabs(x) * s1) * s2);                  // E4M3 subnormal grid
    return c ? c : 1u;            // an underflowed nonzero still rounds up to 2^-9
}

// the 16 codes of a lane (c), squares added to *sq (FAST)
template <bool FAST, bool I8>
__device__ __forceinline__ void cast16(const double (&x)[kCastH], const CastRow& cr, uint32_t (&c)[kCastH],
                                       unsigned long long* sq) {
    bool slow = false;
#pragma unroll
    for (int q = 0; q < kCastH; ++q) {
        const uint32_t hx = static_cast<uint32_t>(__double2hiint(x[q])) & 0x7FFFFFFFu;
        const uint32_t lx = static_cast<uint32_t>(__double2loint(x[q]));
        c[q] = cast_code(hx, lx, cr.add);
        slow |= I8 || hx < cr.thr;
    }
    if (slow) {
#pragma unroll
        for (int q = 0; q < kCastH; ++q) {
            const uint32_t hx = static_cast<uint32_t>(__double2hiint(x[q])) & 0x7FFFFFFFu;
            if (I8 || hx < cr.thr) c[q] = cast_code_slow<I8>(x[q], cr);
        }
    }
    if (FAST) {
        unsigned long long s = 0;
#pragma unroll
        for (int q = 0; q < kCastH; ++q) s += I8 ? static_cast<unsigned long long>(c[q] * c[q]) : fp8_sq_units(c[q]);
        *sq += s;
    }
}

template <bool KMAJOR, bool FAST, bool I8, bool VEC>
__global__ void __launch_bounds__(256) k_cast(const double* __restrict__ X, int64_t rows, int64_t k,
                                              int64_t ld, const unsigned long long* __restrict__ maxbits,
                                              int32_t* __restrict__ eprime, uint8_t* __restrict__ xbar,
                                              int gplanes, int64_t k_pad,
                                              int32_t* __restrict__ status,
                                              unsigned long long* __restrict__ sumsq) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    // MN-major: the lane's row, its 16 consecutive k from h; K-major: the warp's row, the
    // lane's 8 pairs of consecutive k at h + 64 j (each 16-byte load of the warp is one
    // coalesced 512-byte run, each 2-byte store one 64-byte run)
    int64_t r, h;
    if (!KMAJOR) {
        r = static_cast<int64_t>(blockIdx.x) * 32 + lane;
        h = static_cast<int64_t>(blockIdx.y) * TH + w * kCastH;
    } else {
        r = static_cast<int64_t>(blockIdx.x) * 8 + w;
        h = static_cast<int64_t>(blockIdx.y) * (32 * kCastH) + 2 * lane;
    }
    const unsigned long long mb = (r < rows) ? maxbits[r] : 0ull;
    const CastRow cr = cast_row<I8>(mb);
    if (blockIdx.y == 0 && (KMAJOR ? lane == 0 : w == 0) && r < rows) {
        eprime[r] = cr.e;
        if (cr.bad) atomicOr(status, 1);
    }
    double x[kCastH];
    if (!KMAJOR) {
        const double* p = X + r + h * ld;
        if (r < rows && h + kCastH <= k) {
#pragma unroll
            for (int q = 0; q < kCastH; ++q) x[q] = __ldg(p + q * ld);
        } else {
#pragma unroll
            for (int q = 0; q < kCastH; ++q) x[q] = (r < rows && h + q < k) ? __ldg(p + q * ld) : 0.0;
        }
    } else {
        const double* p = X + r * ld + h;
        if (VEC && r < rows && h + 64 * (kCastH / 2 - 1) + 2 <= k) {
#pragma unroll
            for (int j = 0; j < kCastH / 2; ++j) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(p + 64 * j));
                x[2 * j] = v.x;
                x[2 * j + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kCastH / 2; ++j) {
                const int64_t hj = h + 64 * j;
                x[2 * j] = (r < rows && hj < k) ? __ldg(p + 64 * j) : 0.0;
                x[2 * j + 1] = (r < rows && hj + 1 < k) ? __ldg(p + 64 * j + 1) : 0.0;
            }
        }
    }
    unsigned long long sq = 0;
    uint32_t c[kCastH];
    cast16<FAST, I8>(x, cr, c, &sq);
    if (FAST) {
        if (KMAJOR) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
            if (lane == 0 && sq && r < rows) atomicAdd(sumsq + r, sq);
        } else {
            // the 8 warps share the block's 32 rows: one atomic per row and block
            __shared__ unsigned long long part[8][32];
            part[w][lane] = sq;
            __syncthreads();
            if (w == 0) {
#pragma unroll
                for (int v = 1; v < 8; ++v) sq += part[v][lane];
                if (sq && r < rows) atomicAdd(sumsq + r, sq);
            }
        }
    } else if (!KMAJOR) {
        // 16 codes of one 128-byte chunk (h mod 128 is a multiple of 16), padding included:
        // the buffer is reused across calls
        uint4 word;
        word.x = c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24);
        word.y = c[4] | (c[5] << 8) | (c[6] << 16) | (c[7] << 24);
        word.z = c[8] | (c[9] << 8) | (c[10] << 16) | (c[11] << 24);
        word.w = c[12] | (c[13] << 8) | (c[14] << 16) | (c[15] << 24);
        *reinterpret_cast<uint4*>(xbar + chunk_offset(r, static_cast<uint32_t>(h / TH), gplanes, k_pad) + (h % TH)) =
            word;
    } else {
#pragma unroll
        for (int j = 0; j < kCastH / 2; ++j) {
            const int64_t hj = h + 64 * j;      // up to round_up(k, 512) <= k_pad (padding: zero codes)
            *reinterpret_cast<uint16_t*>(xbar + chunk_offset(r, static_cast<uint32_t>(hj / TH), gplanes, k_pad) +
                                         (hj % TH)) = static_cast<uint16_t>(c[2 * j] | (c[2 * j + 1] << 8));
        }
    }
}

// ---------------------------------------------------------------------------------
// One-read prescale (accurate mode): step 1 needs the row maximum before it can cast, so
// the plain form reads X twice (k_rowmax, then k_cast).  Here X is read once:
//   k_cast_local  casts every 128-wide chunk of a row with the chunk's own exponent
//                 e_loc = 7 - floor(log2 max_chunk|x|) >= e' (codes RU_e4m3(|x| 2^e_loc)),
//                 records e_loc and merges the chunk maximum into the row maximum;
//   k_rescale     then moves each chunk to the row exponent: code <- RU_e4m3(v 2^-d),
//                 d = e_loc - e' >= 0, touching only chunks with d > 0.
// Exact: both roundings are upward and the row-scale E4M3 grid {i 2^q : i < 16, q >= -9}
// is a subset of the chunk grid scaled by 2^-d ({i 2^q : q >= -9-d}) wherever the values
// live (< 2^(8-d)), so RU_row(RU_chunk(y)) = RU_row(y) -- the same A-bar as k_cast,
// bit for bit (tests).  INT8 (R16): ceil(ceil(y) / 2^d) = ceil(y / 2^d).
constexpr int16_t kZeroChunk = 32767;      // e_loc of an all-zero chunk (nothing to rescale)

template <bool KMAJOR, bool I8>
__global__ void __launch_bounds__(256) k_cast_local(const double* __restrict__ X, int64_t rows, int64_t k,
                                                    int64_t ld, unsigned long long* __restrict__ maxbits,
                                                    int16_t* __restrict__ eloc, int64_t kc,
                                                    uint8_t* __restrict__ xbar, int gplanes, int64_t k_pad) {
    __shared__ double tile[TR * TP];
    const int64_t h0 = static_cast<int64_t>(blockIdx.x) * TH;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * TR;
    load_tile<KMAJOR>(X, rows, k, ld, r0, h0, tile);
    __syncthreads();
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
    for (int j = 0; j < TR / 8; ++j) {
        const int rr = w + 8 * j;
        const int64_t r = r0 + rr;
        double x[4];
        unsigned long long mx = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            x[q] = tile[rr * TP + lane * 4 + q];
            const unsigned long long b = __double_as_longlong(fabs(x[q]));
            mx = b > mx ? b : mx;
        }
        {   // warp max of the 64-bit patterns: high words, then low words among the leaders
            const uint32_t hi = static_cast<uint32_t>(mx >> 32);
            const uint32_t hmax = __reduce_max_sync(0xffffffffu, hi);
            const uint32_t lmax = __reduce_max_sync(0xffffffffu, hi == hmax ? static_cast<uint32_t>(mx) : 0u);
            mx = (static_cast<unsigned long long>(hmax) << 32) | lmax;
        }
        const int e = eprime_of<I8>(mx);
        if (lane == 0 && r < rows) {
            if (mx) atomicMax(maxbits + r, mx);
            eloc[r * kc + blockIdx.x] = mx ? static_cast<int16_t>(e) : kZeroChunk;
        }
        const double s1 = pow2d(e >> 1), s2 = pow2d(e - (e >> 1));
        uint32_t word = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t c = 0;
            if (x[q] != 0.0 && mx < 0x7FF0000000000000ull) {
                if (I8) {
                    c = static_cast<uint32_t>(ceil((fabs(x[q]) * s1) * s2));
                } else {
                    const uint32_t hx = static_cast<uint32_t>(__double2hiint(x[q])) & 0x7FFFFFFFu;
                    const uint32_t lx = static_cast<uint32_t>(__double2loint(x[q]));
                    const int ey = static_cast<int>(hx >> 20) + e;
                    if ((hx >> 20) != 0u && ey >= 1017) {
                        const uint32_t hy = hx + (static_cast<uint32_t>(e) << 20);
                        const uint32_t sticky = ((hy & 0x1FFFFu) | lx) != 0u ? 0x20000u : 0u;
                        c = (((hy & ~0x1FFFFu) + sticky) >> 17) - 8128u;
                    } else {
                        c = fp8_ru_code((fabs(x[q]) * s1) * s2);
                        c = c ? c : 1u;
                    }
                }
            }
            word |= c << (8 * q);
        }
        // padding rows too (zero codes): the buffer is reused across calls
        *reinterpret_cast<uint32_t*>(xbar + chunk_offset(r, blockIdx.x, gplanes, k_pad) + lane * 4) = word;
    }
}

// one E4M3 code (non-negative) of value v -> RU_e4m3(v 2^-d), d >= 1
__device__ __forceinline__ uint32_t fp8_code_shift_ru(uint32_t c, int d) {
    const uint32_t E = c >> 3, M = c & 7u;
    if (static_cast<int>(E) > d) return c - (static_cast<uint32_t>(d) << 3);   // stays normal: exact
    if (c == 0u) return 0u;
    if (d >= 16) return 1u;                                       // below 2^-9: the smallest subnormal
    const uint32_t v = E ? (8u + M) << (E - 1u) : M;              // value in units of 2^-9 (< 2^15)
    return (v + (1u << d) - 1u) >> d;                             // ceil, a subnormal code 1..8
}

// Warp per row and 32-chunk range (blockIdx.x), 8 rows per block (grid-stride over row
// groups); each lane moves 16 bytes, so one pass of the warp covers 4 chunks (512 B) and
// the 8 passes are independent (loads in flight together).  The row's exponent is read once.
template <bool I8>
__global__ void __launch_bounds__(256) k_rescale(int64_t rows, const unsigned long long* __restrict__ maxbits,
                                                 const int16_t* __restrict__ eloc, int64_t kc,
                                                 int32_t* __restrict__ eprime, int32_t* __restrict__ status,
                                                 uint8_t* __restrict__ xbar, int gplanes, int64_t k_pad) {
    const int lane = threadIdx.x & 31;
    const uint32_t c0 = blockIdx.x * 32u;
    for (int64_t r = static_cast<int64_t>(blockIdx.y) * 8 + (threadIdx.x >> 5); r < rows;
         r += static_cast<int64_t>(gridDim.y) * 8) {
        const unsigned long long mb = maxbits[r];
        const int ep = eprime_of<I8>(mb);
        const bool bad = mb >= 0x7FF0000000000000ull;             // NaN / Inf row: zero bounds (R12)
        if (c0 == 0 && lane == 0) {
            eprime[r] = ep;
            if (bad) atomicOr(status, 1);
        }
#pragma unroll 4
        for (int it = 0; it < 8; ++it) {
            const uint32_t c = c0 + it * 4 + (lane >> 3);
            if (c >= kc) break;
            const int el = eloc[r * kc + c];
            if (el == kZeroChunk) continue;                       // zero chunk: codes are 0 already
            const int d = el - ep;
            if (d == 0 && !bad) continue;
            uint4* p = reinterpret_cast<uint4*>(xbar + chunk_offset(r, c, gplanes, k_pad) + (lane & 7) * 16);
            if (bad) { *p = make_uint4(0u, 0u, 0u, 0u); continue; }
            uint4 w = *p;
            uint32_t* wv = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                uint32_t o = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t b = (wv[t] >> (8 * q)) & 0xFFu;
                    const uint32_t nb = I8 ? (d >= 8 ? (b ? 1u : 0u) : (b + (1u << d) - 1u) >> d)
                                           : fp8_code_shift_ru(b, d);
                    o |= nb << (8 * q);
                }
                wv[t] = o;
            }
            *p = w;
        }
    }
}


// ---------------------------------------------------------------------------------
// k_exps: scaling exponents from the bound maxima (eq. mu-computation)

__global__ void k_exps(const unsigned long long* __restrict__ maxbits,
                       const int32_t* __restrict__ eprime, const uint32_t* __restrict__ rsmax,
                       int64_t count, ExpParams ep, int32_t* __restrict__ e_out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= count) return;
    const unsigned long long mb = maxbits[r];
    if (mb == 0ull) { e_out[r] = 0; return; }               // zero row (R3)
    if (mb >= 0x7FF0000000000000ull) { e_out[r] = kExpNonFinite; return; }   // NaN / Inf (R12)
    const float R = __uint_as_float(rsmax[r]);
    if (!(R > 0.0f)) { e_out[r] = eprime[r]; return; }       // no nonzero product
    const float cbar = __fmul_ru(ep.f_k, R);                 // RU(f_k C-bar') (eq. barCupper, R5)
    const float x1 = __double2float_rd(log2(static_cast<double>(cbar)));   // R7
    const float x2 = __fmul_rd(ep.delta, x1);
    const float x3 = __fadd_rd(ep.p_prime, x2);
    e_out[r] = eprime[r] + static_cast<int>(floorf(x3));   // int() = floor (R8)
}

// ---------------------------------------------------------------------------------
// k_exps_fast: fast-mode exponents (reading R15)
//   log2 mu_r = e'_r + t_r,  t_r = max{t : 2^(2t) S_r <= H},  H = h 2^th = RD64((P-1)/2)
// decided exactly in integers: with S_r = U 2^-us (us = 18: FP8 squares) the test is
// U <= h 2^d, d = th + us - 2t.

__device__ __forceinline__ bool fast_fits(unsigned long long U, unsigned long long h, int hbits, int d) {
    if (d >= 0) return hbits + d > 63 || U <= (h << d);
    return -d < 64 && U <= (h >> -d);
}

// The same rule serves the INT8 scheme (R16) with U = R_r (exact bound-GEMM row max,
// `u32`) or U = sum of squares (fast), both in units of 1 (ushift = 0).
__global__ void k_exps_fast(const unsigned long long* __restrict__ maxbits,
                            const int32_t* __restrict__ eprime,
                            const unsigned long long* __restrict__ sumsq,
                            const uint32_t* __restrict__ u32, int64_t count,
                            FastExpParams fp, int ushift, int32_t* __restrict__ e_out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= count) return;
    const unsigned long long U = sumsq ? sumsq[r] : static_cast<unsigned long long>(u32[r]);
    if (maxbits[r] == 0ull) { e_out[r] = 0; return; }       // zero row (R3)
    if (maxbits[r] >= 0x7FF0000000000000ull) { e_out[r] = kExpNonFinite; return; }   // R12
    if (U == 0ull) { e_out[r] = eprime[r]; return; }        // no nonzero product (R3)
    const int hbits = 64 - __clzll(static_cast<long long>(fp.h));
    const int ubits = 64 - __clzll(static_cast<long long>(U));
    // U < 2^ubits <= h 2^(ubits - hbits + 1): start one step above the answer
    int t = (fp.th + ushift - (ubits - hbits + 1)) / 2 + 2;
    while (!fast_fits(U, fp.h, hbits, fp.th + ushift - 2 * t)) --t;
    e_out[r] = eprime[r] + t;
}

// ---------------------------------------------------------------------------------
// k_digits: X' = trunc(2^e x) (exact), r_l = mod(X', p_l), FP8 digits
//
// Arithmetic is arranged to stay on the FP64/FP32/INT pipes (no conversion-pipe
// instructions except the final E4M3 packing):
//   * 2^e scaling by two exact power-of-two multiplies, truncation by an RZ add of 2^52;
//   * q = round(M/p) by fma(M, 1/p, 1.5*2^52) - 1.5*2^52, r = fma(-q, p, M) exact,
//     and r read as an int from the low word of r + 1.5*2^52;
//   * int -> float by the 1.5*2^23 bit trick, round / ceil of r/s by magic adds.

__device__ __forceinline__ float i2f_small(int v) {       // exact for |v| < 2^22
    return __int_as_float(0x4B400000 + v) - 12582912.0f;
}
constexpr double kMagic52 = 6755399441055744.0;           // 1.5 * 2^52
constexpr float kMagic23 = 12582912.0f;                   // 1.5 * 2^23

__device__ __forceinline__ double dfma_rn(double a, double b, double c) {   // keeps b, c in registers
    double d;
    asm("fma.rn.f64 %0, %1, %2, %3;" : "=d"(d) : "d"(a), "d"(b), "d"(c));
    return d;
}

// k_digits: each lane handles kEPL consecutive elements of a row and stores kEPL bytes per
// digit plane (kEPL = 8 -- one 8-byte store per plane -- was measured: 4 % fewer
// instructions but 17 % slower for the MN-major operand, 78 vs 50 registers)
constexpr int kEPL = 4;
using DWord = uint32_t;          // kEPL bytes of one digit plane
static_assert(sizeof(DWord) == kEPL && TH % kEPL == 0 && 32 % (TH / kEPL) == 0, "k_digits lane map");

// residue and digits of one modulus for the kEPL elements of a lane; NSTEP = 1: |y| < 2^50 p_min
// (~2^59 for the hybrid moduli), NSTEP = 2: |y| < 2^86 p_min (first reduced modulo
// Q = p 2^36, exactly), NSTEP = 0: the general M 2^E form with (2^E mod p) from the
// table (any |y|).  The limits keep every rounding quotient below 2^51, where the
// 1.5 2^52 magic-number rounding is exact.
// SQ: 1 square, 0 non-square, -1 read md.square at run time, 2 INT8 scheme (the residue
// itself, as a two's-complement byte, is the single operand plane of the modulus)
template <int SQ>
__device__ __forceinline__ void emit_digits(const ModDig& md, const float (&rf)[kEPL], uint8_t* o, int pitch);

template <int NSTEP, int SQ>
__device__ __forceinline__ void digits_one_modulus(const ModDig& md, int l, int plane0, const double (&y)[kEPL],
                                                   const double (&M)[kEPL], const int (&E)[kEPL],
                                                   const uint16_t* __restrict__ pow2tab,
                                                   uint8_t* out, int pitch) {
    const double pinv = md.pinv_d, pd = md.p_d, magic = kMagic52;
    float rf[kEPL];
#pragma unroll
    for (int q = 0; q < kEPL; ++q) {
        int ri;
        if (NSTEP == 0) {
            const double qq = dfma_rn(M[q], pinv, magic) - magic;
            const double rd = fma(-qq, pd, M[q]);
            ri = __double2loint(rd + magic);
            const int tw = __ldg(pow2tab + l * kPow2Tab + min(E[q], kPow2Tab - 1));
            const float v = i2f_small(ri * tw);                           // |.| < 2^21
            const float qv = fmaf(v, md.pinv_f, kMagic23) - kMagic23;
            ri = __float_as_int(fmaf(-qv, md.p_f, v) + kMagic23) - 0x4B400000;
            if (y[q] < 0.0) ri = -ri;
        } else {
            double yy = y[q];
            if (NSTEP == 2) {
                const double Q = pd * 68719476736.0, Qinv = pinv * (1.0 / 68719476736.0);  // p 2^36
                const double q1 = dfma_rn(yy, Qinv, magic) - magic;
                yy = fma(-q1, Q, yy);                                     // exact, |yy| < 1.5 Q
            }
            const double qq = dfma_rn(yy, pinv, magic) - magic;           // round(y/p) (+-1)
            const double rd = fma(-qq, pd, yy);                           // exact, |rd| < 1.5 p
            ri = __double2loint(rd + magic);
        }
        rf[q] = __int_as_float(0x4B400000 + ri);                          // r + 1.5 2^23
    }
    // exact symmetric range [-floor(p/2), ceil(p/2)-1] (R2) in packed FP32:
    // r <- r - p round((r + h)/p), h = 0 (odd p) or 1/2 (even p): no ties can occur
    {
        const float2 M2 = make_float2(kMagic23, kMagic23), nM2 = make_float2(-kMagic23, -kMagic23);
        const float2 pi2 = make_float2(md.pinv_f, md.pinv_f), hp2 = make_float2(md.hp_f, md.hp_f);
        const float2 np2 = make_float2(-md.p_f, -md.p_f);
#pragma unroll
        for (int q = 0; q < kEPL; q += 2) {
            const float2 r = __fadd2_rn(make_float2(rf[q], rf[q + 1]), nM2);
            const float2 qv = __fadd2_rn(__fadd2_rn(__ffma2_rn(r, pi2, hp2), M2), nM2);
            const float2 rs = __ffma2_rn(qv, np2, r);
            rf[q] = rs.x;
            rf[q + 1] = rs.y;
        }
    }
    emit_digits<SQ>(md, rf, out + plane0 * pitch, pitch);
}

// the digit planes (or the INT8 residue plane) of one modulus from the exact symmetric
// residues rf[kEPL] of the lane's kEPL consecutive elements; `pitch` = bytes between planes
template <int SQ>
__device__ __forceinline__ void emit_digits(const ModDig& md, const float (&rf)[kEPL], uint8_t* o, int pitch) {
    if (SQ == 2) {
        DWord w = 0;
#pragma unroll
        for (int q = 0; q < kEPL; ++q)
            w |= static_cast<DWord>((static_cast<uint32_t>(__float_as_int(rf[q] + kMagic23) - 0x4B400000) & 0xFFu))
                 << (8 * q);
        *reinterpret_cast<DWord*>(o) = w;
        return;
    }
    // digit arithmetic on packed FP32 pairs (sm_100 FFMA2/FADD2); every value is an exact
    // small integer, the magic-number adds implement round / ceil
    const float2 M2 = make_float2(kMagic23, kMagic23), nM2 = make_float2(-kMagic23, -kMagic23);
    if (SQ == 1 || (SQ < 0 && md.square)) {
        // D1 = round(r/s) ties-to-even, D2 = r - s D1 (R9)
        const float2 is2 = make_float2(md.inv_s_f, md.inv_s_f), ns2 = make_float2(-md.s_f, -md.s_f);
        DWord w1 = 0, w2 = 0;
#pragma unroll
        for (int q = 0; q < kEPL; q += 2) {
            const float2 r = make_float2(rf[q], rf[q + 1]);
            const float2 d1 = __fadd2_rn(__ffma2_rn(r, is2, M2), nM2);
            const float2 d2 = __ffma2_rn(d1, ns2, r);
            w1 |= static_cast<DWord>(cvt_e4m3x2(d1.x, d1.y)) << (8 * q);
            w2 |= static_cast<DWord>(cvt_e4m3x2(d2.x, d2.y)) << (8 * q);
        }
        *reinterpret_cast<DWord*>(o) = w1;
        *reinterpret_cast<DWord*>(o + pitch) = w2;
    } else {
        // D1 = sign(r) ceil(|r|/16), D2 = r - 16 D1, D3 = D1 + D2
        const float2 s16 = make_float2(0.0625f, 0.0625f), n16 = make_float2(-16.0f, -16.0f);
        DWord w1 = 0, w2 = 0, w3 = 0;
#pragma unroll
        for (int q = 0; q < kEPL; q += 2) {
            const float2 r = make_float2(rf[q], rf[q + 1]);
            const float2 a = make_float2(fabsf(rf[q]), fabsf(rf[q + 1]));
            const float2 c = __fadd2_rn(__ffma2_ru(a, s16, M2), nM2);          // ceil(|r|/16)
            const float2 d1 = make_float2(copysignf(c.x, r.x), copysignf(c.y, r.y));
            const float2 d2 = __ffma2_rn(d1, n16, r);
            const float2 d3 = __fadd2_rn(d1, d2);
            w1 |= static_cast<DWord>(cvt_e4m3x2(d1.x, d1.y)) << (8 * q);
            w2 |= static_cast<DWord>(cvt_e4m3x2(d2.x, d2.y)) << (8 * q);
            w3 |= static_cast<DWord>(cvt_e4m3x2(d3.x, d3.y)) << (8 * q);
        }
        *reinterpret_cast<DWord*>(o) = w1;
        *reinterpret_cast<DWord*>(o + pitch) = w2;
        *reinterpret_cast<DWord*>(o + 2 * pitch) = w3;
    }
}

template <int NSTEP, int NMOD, bool I8, int NSQ>
__device__ __forceinline__ void digits_all_moduli(const DigitParams& dp, const double (&y)[kEPL],
                                                  const double (&M)[kEPL], const int (&E)[kEPL],
                                                  uint8_t* out, int pitch) {
    if (I8) {
        // INT8 scheme: one S8 plane per modulus, plane l
        if (NMOD > 0) {
#pragma unroll
            for (int l = 0; l < NMOD; ++l)
                digits_one_modulus<NSTEP, 2>(dp.mod[l], l, l, y, M, E, dp.pow2tab, out, pitch);
        } else {
#pragma unroll 1
            for (int l = 0; l < dp.num_moduli; ++l)
                digits_one_modulus<NSTEP, 2>(dp.mod[l], l, l, y, M, E, dp.pow2tab, out, pitch);
        }
    } else if (NMOD > 0) {
        // hybrid order (eq. p_list_hybrid): the first min(N, 6) moduli are the squares;
        // Karatsuba family (eq. p_list_karatsuba, NSQ = 0): none
#pragma unroll
        for (int l = 0; l < NMOD && l < NSQ; ++l)
            digits_one_modulus<NSTEP, 1>(dp.mod[l], l, 2 * l, y, M, E, dp.pow2tab, out, pitch);
#pragma unroll
        for (int l = NSQ; l < NMOD; ++l)
            digits_one_modulus<NSTEP, 0>(dp.mod[l], l, 2 * NSQ + 3 * (l - NSQ), y, M, E,
                                         dp.pow2tab, out, pitch);
    } else {
#pragma unroll 1
        for (int l = 0; l < dp.num_moduli; ++l)
            digits_one_modulus<NSTEP, -1>(dp.mod[l], l, dp.mod[l].plane0, y, M, E, dp.pow2tab, out, pitch);
    }
}

// The common case |X'| < 2^50 p_min with the moduli taken in pairs: ONE FP64 reduction
// modulo Q = p_l p_(l+1) (< 2^21; Q = p_l for a last odd one out) -- |y/Q| < 2^50, so the
// magic-number quotient is round(y/Q) of an argument within 2^-3 of y/Q and
// |r_Q| = |y - qQ| < Q (1/2 + 2^-3) < 2^21 is exact -- then each modulus' symmetric residue
// (R2) in ONE FP32 step r = r_Q - p rint((r_Q + h)/p), h = 1/2 for the even modulus (index
// EVEN), else 0: the computed quotient is within 2^-3/p of (r_Q + h)/p, which is never
// closer than 1/(2p) to a half-integer, so the rounding is exact.  Bit-identical to
// digits_one_modulus<1, .> (same residues, same digit code).
template <int NMOD, bool I8, int NSQ, int EVEN>
__device__ __forceinline__ void digits_paired(const DigitParams& dp, const double (&y)[kEPL], uint8_t* out, int pitch) {
    const float2 M2 = make_float2(kMagic23, kMagic23), nM2 = make_float2(-kMagic23, -kMagic23);
#pragma unroll
    for (int l = 0; l < NMOD; l += 2) {
        const double Q = dp.mod[l].q2_d, Qi = dp.mod[l].q2inv_d, magic = kMagic52;
        float rq[kEPL];
#pragma unroll
        for (int q = 0; q < kEPL; ++q) {
            const double qq = dfma_rn(y[q], Qi, magic) - magic;
            const double rd = fma(-qq, Q, y[q]);                             // exact, |rd| < 2^21
            rq[q] = __int_as_float(0x4B400000 + __double2loint(rd + magic));  // r_Q + 1.5 2^23
        }
        float2 r2[kEPL / 2];
#pragma unroll
        for (int q = 0; q < kEPL; q += 2) r2[q / 2] = __fadd2_rn(make_float2(rq[q], rq[q + 1]), nM2);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int lm = l + u;
            if (lm >= NMOD) break;
            const ModDig& md = dp.mod[lm];
            const float2 pi2 = make_float2(md.pinv_f, md.pinv_f), np2 = make_float2(-md.p_f, -md.p_f);
            float rf[kEPL];
#pragma unroll
            for (int q = 0; q < kEPL; q += 2) {
                const float2 x = (lm == EVEN) ? __fadd2_rn(r2[q / 2], make_float2(0.5f, 0.5f)) : r2[q / 2];
                const float2 qv = __fadd2_rn(__ffma2_rn(x, pi2, M2), nM2);
                const float2 sv = __ffma2_rn(qv, np2, r2[q / 2]);
                rf[q] = sv.x;
                rf[q + 1] = sv.y;
            }
            if (I8) {
                emit_digits<2>(md, rf, out + lm * pitch, pitch);
            } else if (lm < NSQ) {
                emit_digits<1>(md, rf, out + 2 * lm * pitch, pitch);
            } else {
                emit_digits<0>(md, rf, out + (2 * NSQ + 3 * (lm - NSQ)) * pitch, pitch);
            }
        }
    }
}

// SUP: the super-chunk is kSuper bytes (k_pad >= kSuper), so plane offsets are immediates;
// otherwise S = k_pad (< kSuper, one super-chunk per row), a run-time pitch.
template <bool KMAJOR, int NMOD, bool I8, int NSQ, bool SUP>
__global__ void __launch_bounds__(256, 6) k_digits(const double* __restrict__ X, int64_t rows,
                                                int64_t k, int64_t ld,
                                                const int32_t* __restrict__ e_scale,
                                                const unsigned long long* __restrict__ maxbits,
                                                const __grid_constant__ DigitParams dp,
                                                uint8_t* __restrict__ planes, int64_t rows_pad,
                                                int64_t k_pad) {
    __shared__ double tile[TR * TP];
    const int64_t h0 = static_cast<int64_t>(blockIdx.x) * TH;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * TR;
    load_tile<KMAJOR>(X, rows, k, ld, r0, h0, tile);
    __syncthreads();
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    // plane pitch 128 S: a compile-time immediate for S = kSuper
    const int pitch = kRowBlk * (SUP ? kSuper : static_cast<int>(k_pad));
    // a lane owns kEPL consecutive k of one row: kLPR lanes per row, 32 / kLPR rows per warp
    constexpr int kLPR = TH / kEPL, kRPW = 32 / kLPR;
    static_assert(kRPW == 1, "one row per warp: the per-row path choice below is warp-uniform");
    const int lrow = lane / kLPR, hl = (lane % kLPR) * kEPL;
    // the block's 32 rows lie in one 128-row block of the layout (TR divides kRowBlk), so a
    // row's slab offset is the tile's plus rr S (row stride S inside a plane slab)
    static_assert(kRowBlk % TR == 0, "a conversion tile must not straddle 128-row blocks");
    uint8_t* const out0 = planes + chunk_offset_planes<SUP>(r0, blockIdx.x, dp.num_planes, k_pad) + hl;
    const int row_stride = SUP ? kSuper : static_cast<int>(k_pad);
    const int rows_i = static_cast<int>(rows), r0i = static_cast<int>(r0);   // rows < 2^21 (kMaxRows)
#pragma unroll 1
    for (int j = 0; j < TR / (8 * kRPW); ++j) {
        const int rr = (j * 8 + w) * kRPW + lrow;
        const int r = r0i + rr;
        int e = (r < rows_i) ? e_scale[r] : 0;
        if (e == kExpNonFinite) e = 0;                    // NaN / Inf row: C gets NaN (R12)
        // plane x of this (row, super-chunk) at out + x S: immediate store offsets (SUP)
        uint8_t* out = out0 + rr * row_stride;
        // Common case, decided per row from step 1's row maximum: |X'| < 2^52 and 2^e a
        // normal double.  Then trunc(x 2^e) is ONE fused multiply-add rounded toward zero,
        // fma.rz(x, 2^e, +-2^52) - (+-2^52) with the sign of x (|x 2^e| + 2^52 lies in
        // [2^52, 2^53) where the ulp is 1), and |X'| < 2^52 < lim1 admits the paired residues.
        {
            const unsigned long long mb = !maxbits ? ~0ull : (r < rows_i ? maxbits[r] : 0ull);   // padding rows: zero
            const bool fast = mb == 0ull || (mb < 0x7FF0000000000000ull && e >= -1022 && e <= 1023 &&
                                             ilog2_bits(mb) + e <= 51);
            if (fast && NMOD > 0) {
                const double sc2 = pow2d(e);
                double y[kEPL];
#pragma unroll
                for (int q = 0; q < kEPL; ++q) {
                    const double x = tile[rr * TP + hl + q];
                    const double m52 = __hiloint2double((__double2hiint(x) & 0x80000000) | 0x43300000, 0);
                    double t;
                    asm("fma.rz.f64 %0, %1, %2, %3;" : "=d"(t) : "d"(x), "d"(sc2), "d"(m52));
                    y[q] = t - m52;                                                // exact (eq. def:A')
                }
                digits_paired<NMOD, I8, NSQ, I8 ? 0 : 1>(dp, y, out, pitch);
                continue;
            }
        }
        double y[kEPL], M[kEPL];
        int E[kEPL];
        // X' = trunc(2^e x) (eq. def:A'): the scaling is exact (one multiply when 2^e is a
        // normal double -- warp-uniform, the warp holds one row -- else two), the truncation
        // one FRND.F64.TRUNC; the reduction depth is chosen from the largest high word (for
        // non-negative doubles a >= lim iff hi(a) >= hi(lim) when lim's low word is zero, as
        // for lim = 2^50 p_min and 2^86 p_min; otherwise the test is conservative)
        uint32_t amax_hi = 0;
        if (e >= -1022 && e <= 1023) {
            const double sc = pow2d(e);
#pragma unroll
            for (int q = 0; q < kEPL; ++q) y[q] = trunc(tile[rr * TP + hl + q] * sc);
        } else {
            const double s1 = pow2d(e >> 1), s2 = pow2d(e - (e >> 1));
#pragma unroll
            for (int q = 0; q < kEPL; ++q) y[q] = trunc((tile[rr * TP + hl + q] * s1) * s2);
        }
#pragma unroll
        for (int q = 0; q < kEPL; ++q)
            amax_hi = max(amax_hi, static_cast<uint32_t>(__double2hiint(y[q])) & 0x7FFFFFFFu);
        // warp-uniform choice of the reduction depth (a NaN / Inf row takes the deepest path;
        // its entries of C are NaN whatever its digits, R12)
        const bool need2 = __any_sync(0xffffffffu, amax_hi >= static_cast<uint32_t>(__double2hiint(dp.lim1)));
        const bool need0 = __any_sync(0xffffffffu, amax_hi >= static_cast<uint32_t>(__double2hiint(dp.lim2)));
        if (need0) {
            // |X'| = M 2^E with M < 2^53 an integer (E = 0 below 2^53)
#pragma unroll
            for (int q = 0; q < kEPL; ++q) {
                double a = fabs(y[q]);
                int ee = 0;
                if (a >= 9007199254740992.0) {
                    ee = static_cast<int>((__double_as_longlong(a) >> 52) & 0x7FF) - 1023 - 52;
                    a = a * pow2d(-ee);
                }
                M[q] = a;
                E[q] = ee;
            }
            digits_all_moduli<0, NMOD, I8, NSQ>(dp, y, M, E, out, pitch);
        } else if (need2) {
            digits_all_moduli<2, NMOD, I8, NSQ>(dp, y, M, E, out, pitch);
        } else if (NMOD > 0) {
            digits_paired<NMOD, I8, NSQ, I8 ? 0 : 1>(dp, y, out, pitch);   // the even modulus: 256 / 1024 / 512
        } else {
            digits_all_moduli<1, NMOD, I8, NSQ>(dp, y, M, E, out, pitch);
        }
    }
}

__global__ void k_scale(double* C, int64_t m, int64_t n, int64_t ldc, double beta) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
        if (i < m) C[i + j * ldc] = (beta == 0.0) ? 0.0 : beta * C[i + j * ldc];
    }
}

// plane x of the super-chunk layout -> [rows][k] (debug outputs of oz2_dgemm_ex only)
__global__ void k_unpack_plane(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, int gplanes, int x,
                               int64_t rows, int64_t k, int64_t k_pad) {

    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
        for (int64_t h = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; h < k;
             h += static_cast<int64_t>(gridDim.x) * blockDim.x)
            dst[r * k + h] = src[plane_offset(r, h, x, gplanes, k_pad)];
}

// ---------------------------------------------------------------------------------
// launchers

cudaError_t launch_unpack_plane(uint8_t* dst, const uint8_t* src, int gplanes, int x, int64_t rows, int64_t k,
                                int64_t k_pad, cudaStream_t st) {
    if (rows == 0 || k == 0) return cudaSuccess;
    const int64_t gx = (k + 255) / 256;
    dim3 grid(static_cast<unsigned>(gx < 64 ? gx : 64), static_cast<unsigned>(rows < 65535 ? rows : 65535));
    k_unpack_plane<<<grid, 256, 0, st>>>(dst, src, gplanes, x, rows, k, k_pad);
    return cudaGetLastError();
}

cudaError_t launch_rowmax(const double* X, int64_t rows, int64_t k, int64_t ld, bool kmajor,
                          unsigned long long* maxbits, cudaStream_t st) {
    if (rows == 0 || k == 0) return cudaSuccess;
    if (!kmajor) {
        dim3 grid(static_cast<unsigned>((rows + 255) / 256), static_cast<unsigned>((k + 511) / 512));
        k_rowmax<false><<<grid, 256, 0, st>>>(X, rows, k, ld, maxbits);
    } else {
        dim3 grid(static_cast<unsigned>((rows + 7) / 8));
        k_rowmax<true><<<grid, 256, 0, st>>>(X, rows, k, ld, maxbits);
    }
    return cudaGetLastError();
}

cudaError_t launch_cast(const double* X, int64_t rows, int64_t k, int64_t ld, bool kmajor,
                        const unsigned long long* maxbits, int32_t* eprime, uint8_t* xbar, int gplanes,
                        int64_t rows_pad, int64_t k_pad, int32_t* status,
                        unsigned long long* sumsq, bool i8, cudaStream_t st) {
    if (rows_pad == 0 || k == 0) return cudaSuccess;
    // K tiles up to round_up(k, 128) (MN-major) or round_up(k, 512) (K-major, inside k_pad, a
    // multiple of 2048): beyond round_up(k, 128) the layout's padding is never read
    const bool vec = (reinterpret_cast<uintptr_t>(X) & 15u) == 0 && (ld & 1) == 0;
    const dim3 grid = kmajor ? dim3(static_cast<unsigned>(rows_pad / 8), static_cast<unsigned>((k + 511) / 512))
                             : dim3(static_cast<unsigned>(rows_pad / 32), static_cast<unsigned>((k + TH - 1) / TH));
#define OZ2_CAST(KM, FA, I8_, V) k_cast<KM, FA, I8_, V><<<grid, 256, 0, st>>>(X, rows, k, ld, maxbits, eprime, xbar, gplanes, k_pad, status, sumsq)
    const bool fa = sumsq != nullptr;
    if (!kmajor) {
        if (fa) { if (i8) OZ2_CAST(false, true, true, false); else OZ2_CAST(false, true, false, false); }
        else { if (i8) OZ2_CAST(false, false, true, false); else OZ2_CAST(false, false, false, false); }
    } else if (vec) {
        if (fa) { if (i8) OZ2_CAST(true, true, true, true); else OZ2_CAST(true, true, false, true); }
        else { if (i8) OZ2_CAST(true, false, true, true); else OZ2_CAST(true, false, false, true); }
    } else {
        if (fa) { if (i8) OZ2_CAST(true, true, true, false); else OZ2_CAST(true, true, false, false); }
        else { if (i8) OZ2_CAST(true, false, true, false); else OZ2_CAST(true, false, false, false); }
    }
#undef OZ2_CAST
    return cudaGetLastError();
}

cudaError_t launch_cast_local(const double* X, int64_t rows, int64_t k, int64_t ld, bool kmajor,
                              unsigned long long* maxbits, int16_t* eloc, uint8_t* xbar, int gplanes,
                              int64_t rows_pad, int64_t k_pad, bool i8, cudaStream_t st) {
    if (rows == 0 || k == 0) return cudaSuccess;
    const int64_t kc = (k + TH - 1) / TH;
    dim3 grid(static_cast<unsigned>(kc), static_cast<unsigned>(rows_pad / TR));
#define OZ2_CL(KM, I8_) k_cast_local<KM, I8_><<<grid, 256, 0, st>>>(X, rows, k, ld, maxbits, eloc, kc, xbar, gplanes, k_pad)
    if (kmajor) { if (i8) OZ2_CL(true, true); else OZ2_CL(true, false); }
    else { if (i8) OZ2_CL(false, true); else OZ2_CL(false, false); }
#undef OZ2_CL
    return cudaGetLastError();
}

cudaError_t launch_rescale(int64_t rows, int64_t k, const unsigned long long* maxbits, const int16_t* eloc,
                           int32_t* eprime, int32_t* status, uint8_t* xbar, int gplanes, int64_t k_pad, bool i8,
                           cudaStream_t st) {
    if (rows == 0 || k == 0) return cudaSuccess;
    const int64_t kc = (k + TH - 1) / TH, groups = (rows + 7) / 8;   // 8 rows (warps) per block
    dim3 grid(static_cast<unsigned>((kc + 31) / 32), static_cast<unsigned>(groups < 65535 ? groups : 65535));
    if (i8) k_rescale<true><<<grid, 256, 0, st>>>(rows, maxbits, eloc, kc, eprime, status, xbar, gplanes, k_pad);
    else k_rescale<false><<<grid, 256, 0, st>>>(rows, maxbits, eloc, kc, eprime, status, xbar, gplanes, k_pad);
    return cudaGetLastError();
}

cudaError_t launch_exps_fast(const unsigned long long* maxbits, const int32_t* eprime,
                             const unsigned long long* sumsq, const uint32_t* u32, int64_t count,
                             FastExpParams fp, int ushift, int32_t* e_out, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    k_exps_fast<<<static_cast<unsigned>((count + 255) / 256), 256, 0, st>>>(maxbits, eprime, sumsq, u32, count, fp,
                                                                          ushift, e_out);
    return cudaGetLastError();
}

cudaError_t launch_exps(const unsigned long long* maxbits, const int32_t* eprime,
                        const uint32_t* rsmax, int64_t count, ExpParams ep, int32_t* e_out,
                        cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    k_exps<<<static_cast<unsigned>((count + 255) / 256), 256, 0, st>>>(maxbits, eprime, rsmax, count, ep, e_out);
    return cudaGetLastError();
}

cudaError_t launch_digits(const double* X, int64_t rows, int64_t k, int64_t ld, bool kmajor,
                          const int32_t* e, const unsigned long long* maxbits, const DigitParams& dp, uint8_t* planes,
                          int64_t rows_pad, int64_t k_pad, cudaStream_t st) {
    // K tiles up to round_up(k, 128): beyond that the layout's padding is never read
    dim3 grid(static_cast<unsigned>((k + TH - 1) / TH), static_cast<unsigned>(rows_pad / TR));
#define OZ2_DIG_S(NM, I8_, SQ_, SUP)                                                                                    \
    if (kmajor) k_digits<true, NM, I8_, SQ_, SUP><<<grid, 256, 0, st>>>(X, rows, k, ld, e, maxbits, dp, planes, rows_pad, k_pad); \
    else k_digits<false, NM, I8_, SQ_, SUP><<<grid, 256, 0, st>>>(X, rows, k, ld, e, maxbits, dp, planes, rows_pad, k_pad);
#define OZ2_DIG(NM, I8_, SQ_) OZ2_DIG_S(NM, I8_, SQ_, true)
    if (super_bytes(k_pad) != kSuper) {
        // k_pad < kSuper: one super-chunk of k_pad bytes per row, run-time plane pitch (the
        // generic kernels; short-k conversions are a small part of such a call)
        if (dp.int8) { OZ2_DIG_S(0, true, 0, false) }
        else if (dp.num_squares == kNumSquares) { OZ2_DIG_S(0, false, kNumSquares, false) }
        else { OZ2_DIG_S(0, false, 0, false) }
    } else if (dp.even_index != (dp.int8 ? 0 : 1)) {
        // generic (never for the planner's families, whose even modulus is 256 / 1024 / 512)
        if (dp.int8) { OZ2_DIG(0, true, 0) } else { OZ2_DIG(0, false, 0) }
    } else if (dp.int8) {
        switch (dp.num_moduli) {   // INT8 scheme: 14..16 moduli are the FP64-level counts
            case 14: OZ2_DIG(14, true, 0) break;
            case 15: OZ2_DIG(15, true, 0) break;
            case 16: OZ2_DIG(16, true, 0) break;
            default: OZ2_DIG(0, true, 0) break;
        }
    } else if (dp.num_squares == 0 && dp.num_moduli >= 13) {
        switch (dp.num_moduli) {   // Karatsuba family: 13, 14 are the FP64-level counts
            case 13: OZ2_DIG(13, false, 0) break;
            case 14: OZ2_DIG(14, false, 0) break;
            default: OZ2_DIG(0, false, 0) break;
        }
    } else if (dp.num_squares == kNumSquares) {
        switch (dp.num_moduli) {   // hybrid family, fully unrolled for config 2's sweep (12..20)
            case 12: OZ2_DIG(12, false, kNumSquares) break;
            case 13: OZ2_DIG(13, false, kNumSquares) break;
            case 14: OZ2_DIG(14, false, kNumSquares) break;
            case 15: OZ2_DIG(15, false, kNumSquares) break;
            case 16: OZ2_DIG(16, false, kNumSquares) break;
            case 17: OZ2_DIG(17, false, kNumSquares) break;
            case 18: OZ2_DIG(18, false, kNumSquares) break;
            case 19: OZ2_DIG(19, false, kNumSquares) break;
            case 20: OZ2_DIG(20, false, kNumSquares) break;
            default: OZ2_DIG(0, false, kNumSquares) break;
        }
    } else {
        OZ2_DIG(0, false, 0)       // generic: reads md.square per modulus
    }
#undef OZ2_DIG
#undef OZ2_DIG_S
    return cudaGetLastError();
}

cudaError_t launch_scale(double* C, int64_t m, int64_t n, int64_t ldc, double beta, cudaStream_t st) {
    if (m == 0 || n == 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((m + 255) / 256), static_cast<unsigned>(n < 65535 ? n : 65535));
    k_scale<<<grid, 256, 0, st>>>(C, m, n, ldc, beta);
    return cudaGetLastError();
}

}  // namespace oz2
