/*
 * oz2.h -- C ABI of liboz2.so: FP64 GEMM emulated with the Ozaki-II scheme on the
 * FP8 (E4M3 in, FP32 accumulate) tensor cores of an NVIDIA B200 (sm_100a).
 *
 * Method: Uchino, Ozaki, Imamura, "Double-Precision Matrix Multiplication Emulation
 * via Ozaki-II Scheme with FP8 Quantization" (arxiv 2603.10634).  Citations "P:n"
 * are line numbers of that paper's LaTeX source; "Rn" are the readings
 * of silent or ambiguous passages listed in DESIGN.md.
 *
 * Every entry point is extern "C", takes plain pointers and sizes, and returns an
 * int status (0 = success, -i = argument i invalid in BLAS xerbla order, >0 =
 * OZ2_ERR_* runtime failure) unless stated otherwise.  No C++ or torch types cross
 * this boundary.
 */
#ifndef OZ2_H
#define OZ2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------------ */
#define OZ2_SUCCESS            0
#define OZ2_ERR_CUDA           1   /* a CUDA runtime call or kernel launch failed     */
#define OZ2_ERR_ALLOC          2   /* device or pinned host allocation failed         */
#define OZ2_ERR_WORKSPACE      3   /* caller-provided workspace smaller than needed   */
#define OZ2_ERR_NOT_SUPPORTED  4   /* k > 2^22, mixed host/device pointers, no sm_100 */
#define OZ2_ERR_NONFINITE      5   /* oz2_get_status(): A or B held NaN/Inf           */

/* ---- schemes (see oz2_set_scheme) ---------------------------------------------- */
#define OZ2_SCHEME_FP8         0   /* the paper's FP8 Ozaki-II, hybrid moduli (default) */
#define OZ2_SCHEME_INT8        1   /* INT8 Ozaki-II, moduli <= 256 (R16)     */
#define OZ2_SCHEME_FP8_KARATSUBA 2 /* FP8 Ozaki-II, Karatsuba-only moduli   */

/* ---- scaling modes (see oz2_set_mode) ------------------------------- */
#define OZ2_MODE_ACCURATE      0   /* bound GEMM on FP8 tensor cores       */
#define OZ2_MODE_FAST          1   /* Cauchy-Schwarz bound, no bound GEMM (R15)       */

/* ---- the primary call -------------------------------------------------------- */

/*
 * C <- alpha * op(A) op(B) + beta * C, op(A) m x k, op(B) k x n, all FP64,
 * column-major BLAS/cuBLAS conventions (reading R11: the paper states the problem
 * as C ~ AB; alpha, beta, trans and ld follow DGEMM).
 *
 *   transa, transb  'N'/'n' (op(X) = X), 'T'/'t'/'C'/'c' (op(X) = X^T).
 *   m, n, k         >= 0.  The paper assumes k <= 2^16 so that one FP32 accumulation
 *                   of digit products is exact (eq. error-free-FP8-matmult
 *                   P:258-261); longer k (up to 2^22) runs every product in 2^16-long
 *                   K segments whose results are reduced mod p and summed (exact
 *                   modular arithmetic, DESIGN.md NEXT-2); k > 2^22 returns
 *                   OZ2_ERR_NOT_SUPPORTED.
 *   A, lda          A is m x k (transa 'N', lda >= max(1,m)) or k x m (lda >= max(1,k)).
 *   B, ldb          B is k x n (transb 'N', ldb >= max(1,k)) or n x k (ldb >= max(1,n)).
 *   C, ldc          m x n, ldc >= max(1,m).  Read only when beta != 0.
 *   num_moduli      N in [2, 33]: the first N moduli of the hybrid set
 *                   {1089, 1024, 961, 841, 625, 529, 511, 509, ...} (eq. p_list_hybrid,
 *                   P:306-316; P:526 assumes N < 34).  N = 12 is the paper's FP64
 *                   configuration; N = 13 gives FP64-BLAS-level
 *                   error at k = 16384.
 *
 * Pointers may be DEVICE memory (the fast path: everything is enqueued on the
 * library's current stream, see oz2_set_stream, asynchronously; the caller keeps
 * A, B, C alive until the stream work completes) or HOST memory (pageable or
 * pinned; detected with cudaPointerGetAttributes): then A and B are copied to
 * device staging buffers, the same device pipeline runs, C is copied back, and the
 * call returns only after the stream has been synchronised.  All of A, B, C must be
 * of the same kind.
 *
 * Algorithm (accurate mode; workflow P:501-524), all on the device:
 *   1. mu'_i = 2^7/ufp(max_h |a_ih|), A-bar = RU_fp8(|diag(mu') A|); same for B   (eq. def:mu'nu')
 *   2. C-bar' = A-bar B-bar on FP8 tensor cores; keep row/column maxima
 *   3. log2 mu_i = log2 mu'_i + int(P' + delta log2 max_j c-bar_ij)               (eq. mu-computation)
 *   4. A' = trunc(diag(mu) A), residues mod p_l, FP8 digit split
 *   5. 3 exact FP8 GEMMs per modulus, reduced mod p_l in the epilogue             (eqs. 3matmult-notKaratsuba, C'-Karatsuba)
 *   6. C' = mod(sum_l q_l P/p_l C'_l, P) and C = diag(mu)^-1 C' diag(nu)^-1        (eqs. CRT_finalreduction, inversescaling)
 *
 * Fast mode (oz2_set_mode(OZ2_MODE_FAST), Table 2's 3N-GEMM variant) replaces
 * steps 2-3 by the Cauchy-Schwarz bound (reading R15): S_i = sum_h A-bar_ih^2 (exact, from
 * the step-1 FP8 upper bounds, accumulated in integers), log2 mu_i = e'_i + t_i with
 * t_i = max{t : 2^(2t) S_i <= RD64((P-1)/2)}; same for nu.  Steps 4-6 are unchanged.
 *
 * Quick returns (BLAS): m == 0 or n == 0: nothing.  alpha == 0 or k == 0:
 * C <- beta C (C not read when beta == 0).
 * Non-finite entries in A or B: the call still returns 0 (no host sync on the fast
 * path); the device status word is set and oz2_get_status() reports
 * OZ2_ERR_NONFINITE (reading R12).  Every entry of C in a row of op(A) or a column of
 * op(B) holding a NaN or Inf is NaN (its scaling exponent, in the e_mu / e_nu outputs
 * of oz2_dgemm_ex, is INT32_MIN); the other entries are computed normally.
 */
int oz2_dgemm(char transa, char transb, int64_t m, int64_t n, int64_t k,
              double alpha, const double* A, int64_t lda,
              const double* B, int64_t ldb,
              double beta, double* C, int64_t ldc, int num_moduli);

/* ---- extended call: debug outputs and imported exponents ---------------------- */

/*
 * Every pointer field is optional (NULL = not wanted / not given) and must be
 * DEVICE memory.  Outputs are written after the corresponding stage, in the layouts
 * stated; sizes are the caller's responsibility.  Integer exponents are log2 of the
 * power-of-two scaling factors (the paper stores them as INT16; we use int32).
 */
typedef struct oz2_options {
    /* outputs */
    int32_t* e_prime_a;     /* [m]  log2 mu'_i                 (eq. def:mu'nu')          */
    int32_t* e_prime_b;     /* [n]  log2 nu'_j                                            */
    uint8_t* abar;          /* [m][k] row-major E4M3 codes of A-bar (K contiguous)        */
    uint8_t* bbar;          /* [n][k] row-major E4M3 codes of B-bar^T (K contiguous)      */
    float*   rmax;          /* [m]  R_i = max_j C-bar'_ij                    */
    float*   smax;          /* [n]  S_j = max_i C-bar'_ij                    */
    int32_t* e_mu;          /* [m]  log2 mu_i                  (eq. mu-computation)       */
    int32_t* e_nu;          /* [n]  log2 nu_j                  (eq. nu-computation)       */
    uint8_t* digits_a;      /* [M_N][m][k] E4M3 digit planes of A, plane order: per
                               modulus l, x = 1..2 (square) or 1..3 (non-square)          */
    uint8_t* digits_b;      /* [M_N][n][k] same for B^T                                  */
    int16_t* residues;      /* [N][n][m] C'_l (i fastest), symmetric range (R2)          */
    /* inputs */
    const int32_t* e_mu_in; /* [m]  if non-NULL together with e_nu_in: use these scaling */
    const int32_t* e_nu_in; /* [n]  exponents and skip steps 1-3             */
    /* per-call settings (override the thread's oz2_set_mode / oz2_set_scheme /
     * oz2_set_timing for this call only) */
    float*  timing_ms;      /* HOST [7] or NULL: this call's phase times in ms, layout of
                               oz2_get_timing; the call then synchronises its stream      */
    int32_t set_mode;       /* nonzero: run this call in `mode`                           */
    int32_t mode;           /* OZ2_MODE_ACCURATE / OZ2_MODE_FAST                          */
    int32_t set_scheme;     /* nonzero: run this call with `scheme`                       */
    int32_t scheme;         /* OZ2_SCHEME_*                                               */
    int32_t reserved[4];    /* must be zero                                               */
} oz2_options;

int oz2_dgemm_ex(char transa, char transb, int64_t m, int64_t n, int64_t k,
                 double alpha, const double* A, int64_t lda,
                 const double* B, int64_t ldb,
                 double beta, double* C, int64_t ldc, int num_moduli,
                 const oz2_options* opt);

/* ---- runtime state (per host thread) ------------------------------------------ */

/* Stream for subsequent calls from this host thread (cudaStream_t passed as void*;
 * NULL = legacy default stream). */
int oz2_set_stream(void* stream);

/* Scaling mode for subsequent oz2_dgemm / oz2_dgemm_ex calls of this host thread:
 * OZ2_MODE_ACCURATE (default) or OZ2_MODE_FAST; -1 for any other value.  In fast mode
 * the abar/bbar/rmax/smax outputs of oz2_options are not written. */
int oz2_set_mode(int mode);
int oz2_get_mode(void);

/* Scheme for subsequent calls (and host-only queries: oz2_moduli, oz2_plan_query,
 * oz2_workspace_size*) of this host thread.  OZ2_SCHEME_FP8 (default): the paper's method.
 * OZ2_SCHEME_INT8: the INT8 Ozaki-II baseline of the paper's Sec. II on the
 * tcgen05 kind::i8 tensor path -- moduli {256, 255, 253, 251, 247, ...} (eq. p_list), one
 * exact S8 x S8 -> S32 GEMM per modulus (N GEMMs, +1 bound GEMM in accurate mode, Table 2);
 * A-bar = ceil(2^e'|a|) <= 128 (e' = 6 - floor(log2 max|a|)), exact U8 bound GEMM, and
 * log2 mu_i = e'_i + max{t : 2^(2t) R_i <= RD64((P-1)/2)} (reading R16).  k <= 2^16 (else
 * OZ2_ERR_NOT_SUPPORTED).  In oz2_options the abar/bbar outputs then hold the U8 bounds,
 * rmax/smax the exact S32 maxima (as uint32 bits) and digits_a/b the S8 residue planes.
 * OZ2_SCHEME_FP8_KARATSUBA: the FP8 scheme with the Karatsuba-only moduli of the paper's
 * Sec. III-B (eq. p_list_karatsuba: greedy pairwise coprime from 513 down,
 * {513, 512, 511, 509, 505, ...}); every modulus takes the 3-digit Karatsuba split with
 * s = 16 and eq. C'-Karatsuba (3N GEMMs, +1 bound GEMM in accurate
 * mode); FP64 level needs N >= 13.  Everything else (modes, blocking, long K,
 * outputs) is that of OZ2_SCHEME_FP8.
 * Returns -1 for any other value. */
int oz2_set_scheme(int scheme);
int oz2_get_scheme(void);

/* Bytes of device workspace a call with these arguments needs (0 on invalid args). */
size_t oz2_workspace_size(char transa, char transb, int64_t m, int64_t n, int64_t k,
                          int num_moduli);

/* Caller-owned device workspace for subsequent calls from this host thread; the
 * library keeps the pointer (not ownership) until replaced.  ptr == NULL reverts to
 * a library-owned buffer that grows on demand.  Must stay valid until all work
 * enqueued with it has completed.
 *
 * If `bytes` is below oz2_workspace_size(), calls run steps 4-6 on m/n blocks of C that
 * fit (block choice: oz2_plan_blocking), unless oz2_dgemm_ex asks for the
 * whole-problem digit planes or residues.  Steps 1-3 always see the whole problem, so
 * the scaling exponents -- and C, bit for bit -- equal those of the unblocked call. */
int oz2_set_workspace(void* ptr, size_t bytes);

/* m/n blocking (workspace reduction).  oz2_set_blocking forces block sizes
 * (multiples of 256; 0 = automatic) for subsequent calls of this host thread;
 * oz2_get_blocking reports the (mb, nb) the last call used (mb = m, nb = n: unblocked).
 * oz2_workspace_size_blocked gives the bytes for given block sizes (0 = full extent);
 * oz2_plan_blocking picks blocks for a workspace of `bytes` (host only): the largest
 * column block nb (halving from n) admitting a row block mb >= min(m, nb); returns
 * OZ2_ERR_WORKSPACE if not even 256 x 256 blocks fit.  Blocking recomputes A's digits
 * once per column block when mb < m. */
int oz2_set_blocking(int64_t mb, int64_t nb);
int oz2_get_blocking(int64_t* mb, int64_t* nb);
size_t oz2_workspace_size_blocked(int64_t m, int64_t n, int64_t k, int num_moduli,
                                  int64_t mb, int64_t nb);
int oz2_plan_blocking(int64_t m, int64_t n, int64_t k, int num_moduli, size_t bytes,
                      int64_t* mb, int64_t* nb);

/* Synchronises the current stream, returns the device status word of the last call
 * on it (OZ2_SUCCESS or OZ2_ERR_NONFINITE) in *status and clears it. */
int oz2_get_status(int32_t* status);

/* Phase timers (CUDA events on the call's stream).  enable != 0 makes subsequent
 * device-path calls of this host thread record events at the phase boundaries;
 * oz2_get_timing synchronises on the last call's final event and writes up to n
 * floats (ms): [0] prescale (row maxima + A-bar/B-bar cast), [1] bound GEMM,
 * [2] scaling exponents, [3] residue/digit split, [4] residue GEMMs with the
 * modular epilogue (the paper's "gemms" + "requant"), [5] CRT + inverse
 * scaling ("dequant"), [6] total.  Returns OZ2_ERR_NOT_SUPPORTED if the last
 * call recorded no timing. */
int oz2_set_timing(int enable);
int oz2_get_timing(float* ms_out, int n);

/* Frees library-owned buffers and cached plans of this host thread (on every device it
 * used).  A thread that exits without calling it has them freed by its thread-local
 * destructor. */
int oz2_finalize(void);

/* ---- tuning knobs (per host thread; defaults are the measured best) ------------
 *
 * Every setting gives bit-identical results; they only change the kernel schedule.
 * Read at each call (no environment variables are consulted by the library).
 *
 *   OZ2_TUNE_CTA_GROUP   2    residue/bound GEMM tile: 1 = 128x256 single CTA, 2 =
 *                             256x256 CTA pair (tcgen05 cta_group::2), 4 = two pairs
 *                             sharing A by TMA multicast (FP8 kinds; INT8 uses 2)
 *   OZ2_TUNE_SYNC_LEAD   1    progress throttle: chunks a pair may lead the chip-wide
 *                             average (0 = off)
 *   OZ2_TUNE_SYNC_CHUNK  4    k-blocks per throttle chunk (power of two, 1..512)
 *   OZ2_TUNE_L2_PROMO    3    L2 promotion of TMA misses: 0 none, 1 64 B, 2 128 B, 3 256 B
 *   OZ2_TUNE_MAX_UNITS   0    cap on persistent CTA pairs (0 = all; power-wall study)
 *   OZ2_TUNE_TMA_HINT_A  0    L2 policy of A's operand loads: 0 normal, 1 evict-last,
 *   OZ2_TUNE_TMA_HINT_B  0      2 evict-first (same for B)
 *   OZ2_TUNE_MOD_SPLIT  -1    residue-GEMM work items: -1 auto, 0 tile-major, 1 (tile,
 *                             modulus), 2 hybrid (tail wave split)
 *   OZ2_TUNE_FUSED_CRT  -1    CRT in the GEMM epilogue: -1 auto, 0 never, 1 whenever
 *                             the limbs <= 6 and k >= 8192
 *   OZ2_TUNE_SQ_ORDER    1    square-modulus product order: 1 = A1B2, A2B2, A2B1 (L2
 *                             reuse), 0 = the order of eq. 3matmult-notKaratsuba
 *   OZ2_TUNE_CRT_GENERIC 0    1 = the generic standalone CRT kernel (A/B reference)
 *   OZ2_TUNE_HOST_BLOCKS 4    host-pointer calls with pinned C: column blocks of C whose
 *                             device-to-host copies overlap the GEMMs (1 = off)
 *   OZ2_TUNE_KCAT       -1    square moduli: accumulate A1B2 + A2B1 in one TMEM
 *                             accumulator (K-concatenated; two accumulator drains
 *                             instead of three): -1 auto (k <= 2048), 0 off, 1 on (k <= 2^15)
 *   OZ2_TUNE_PRESCALE_2READ 1 accurate-mode step 1: 0 = one read of A and B (chunk-local
 *                             casts, then a rescale of A-bar/B-bar to the row exponent),
 *                             1 = row maxima then cast (two reads; fast mode always)
 *   OZ2_TUNE_EPI_SLEEP 1000   residue GEMM: ns the epilogue warps sleep between polls of a
 *                             filling accumulator (0 = spin on mbarrier.try_wait)
 *   OZ2_TUNE_DIGITS_FMA  0    step 4: rows with |X'| < 2^52 (known from step 1's row maxima)
 *                             scale and truncate with one fma.rz per element (0 = the general
 *                             two-multiply path for every row)
 *   OZ2_TUNE_TILE_N    256    residue-GEMM tile width with CTA pairs (FP8 schemes): 256, or
 *                             512 (256 x 512 tiles: both 256-column TMEM accumulators hold
 *                             one tile, A staged once for both halves)
 *
 * oz2_set_tuning returns -1 for an unknown knob, -2 for a value out of range;
 * oz2_get_tuning writes the current value. */
#define OZ2_TUNE_CTA_GROUP    0
#define OZ2_TUNE_SYNC_LEAD    1
#define OZ2_TUNE_SYNC_CHUNK   2
#define OZ2_TUNE_L2_PROMO     3
#define OZ2_TUNE_MAX_UNITS    4
#define OZ2_TUNE_TMA_HINT_A   5
#define OZ2_TUNE_TMA_HINT_B   6
#define OZ2_TUNE_MOD_SPLIT    7
#define OZ2_TUNE_FUSED_CRT    8
#define OZ2_TUNE_SQ_ORDER     9
#define OZ2_TUNE_CRT_GENERIC 10
#define OZ2_TUNE_HOST_BLOCKS 11
#define OZ2_TUNE_KCAT        12
#define OZ2_TUNE_PRESCALE_2READ 13
#define OZ2_TUNE_EPI_SLEEP   14
#define OZ2_TUNE_DIGITS_FMA  15
#define OZ2_TUNE_TILE_N      16
#define OZ2_TUNE_COUNT       17
int oz2_set_tuning(int knob, int value);
int oz2_get_tuning(int knob, int* value);
void oz2_reset_tuning(void);

/* ---- host-only queries (no device needed) -------------------------------------- */

/* The first num_moduli hybrid moduli (eq. p_list_hybrid). */
int oz2_moduli(int num_moduli, int32_t* p_out);

/* Constants of the plan for (num_moduli, k), for tests and reports. */
typedef struct oz2_plan_info {
    int32_t num_moduli;
    int32_t num_planes;        /* M_N (eq. M)                                   */
    int32_t num_limbs;         /* 32-bit limbs of the CRT integer arithmetic               */
    int32_t num_squares;       /* square moduli among the first N (<= 6)                   */
    float   p_prime;           /* P' = RD32((log2(P-1) - 1)/2)           */
    float   delta;             /* delta = RD32(-1/(2 - 2^-21))           */
    float   f_k;               /* RU32(1/(1 - k 2^-23)), reading R5  (eq. barCupper)       */
    double  log2_P;            /* log2 P                                                   */
    uint32_t P_limbs[12];      /* P, little-endian 32-bit limbs (num_limbs used)           */
    uint32_t w_limbs[33][12];  /* w_l = q_l P/p_l (eq. CRT_finalreduction)                 */
    double  fast_H;            /* RD64((P-1)/2), fast mode's per-side budget (R15)         */
} oz2_plan_info;

int oz2_plan_query(int num_moduli, int64_t k, oz2_plan_info* out);

/* "oz2 <version> sm_100a" */
const char* oz2_version(void);

/* The cudaError_t behind this thread's last OZ2_ERR_CUDA (0 if none yet); its name (e.g.
 * "cudaErrorLaunchOutOfResources") is copied into name_out (cap bytes, NUL-terminated) when
 * name_out is not NULL. */
int oz2_last_cuda_error(char* name_out, int cap);

/* ---- diagnostics ---------------------------------------------------------------- */

/*
 * Raw FP8 GEMM on the same tcgen05 kernel: C32[i][j] = sum_h a[i][h] b[j][h] with
 * E4M3 inputs and the tensor core's FP32 accumulation, for probing the
 * exactness window (eq. error-free-FP8-matmult) and the bound-GEMM rounding (R5).
 * a: [m][k] and b: [n][k] row-major E4M3 codes, device memory, k a multiple of 16;
 * C32: [m][n] row-major float, device memory.  Enqueued on the current stream.
 */
int oz2_fp8_gemm_raw(const uint8_t* a, const uint8_t* b, float* C32,
                     int64_t m, int64_t n, int64_t k);

/* Step 2's kernel on plain operands (the bound GEMM of P:352-362, MODE_BOUND):
 * rmax[i] = max over j and smax[j] = max over i of the FP32 accumulator C32[i][j] =
 * sum_h a[i][h] b[j][h], as float bit patterns merged with atomicMax into the caller's
 * arrays (zero them first; the bit order is the numeric order for non-negative results, as
 * for the RU-cast operands of step 1).  a, b as for oz2_fp8_gemm_raw.  Used to time the
 * tensor-core pipeline with a near-empty epilogue against the vendor FP8 GEMM on the same
 * data (tools/power_probe.py). */
int oz2_fp8_gemm_bound(const uint8_t* a, const uint8_t* b, uint32_t* rmax, uint32_t* smax,
                       int64_t m, int64_t n, int64_t k);

/* The same on the INT8 path (kind::i8): C32[i][j] = sum_h a[i][h] b[j][h], S8 inputs,
 * S32 accumulation (exact while |sum| < 2^31). */
int oz2_int8_gemm_raw(const int8_t* a, const int8_t* b, int32_t* C32,
                      int64_t m, int64_t n, int64_t k);

#ifdef __cplusplus
}
#endif
#endif /* OZ2_H */
