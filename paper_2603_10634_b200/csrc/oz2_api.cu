// oz2_api.cu -- the C ABI (include/oz2.h): argument checking, the host planner
// (moduli, CRT constants, P', delta, f_k), workspace carving, TMA descriptors and the
// launch sequence of the FP8 Ozaki-II pipeline.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/oz2.h"
#include "oz2_internal.h"

namespace oz2 {

// =================================================================================
// host planner: hybrid moduli (eq. p_list_hybrid) and CRT constants
// (eq. CRT_finalreduction) with a small fixed-purpose bigint.

using Big = std::vector<uint32_t>;   // little-endian 32-bit limbs

static void big_trim(Big& a) { while (a.size() > 1 && a.back() == 0) a.pop_back(); }
static void big_mul_small(Big& a, uint32_t s) {
    uint64_t c = 0;
    for (auto& x : a) { const uint64_t v = static_cast<uint64_t>(x) * s + c; x = static_cast<uint32_t>(v); c = v >> 32; }
    if (c) a.push_back(static_cast<uint32_t>(c));
}
static uint32_t big_divmod_small(Big& a, uint32_t s) {
    uint64_t r = 0;
    for (size_t i = a.size(); i-- > 0;) {
        const uint64_t cur = (r << 32) | a[i];
        a[i] = static_cast<uint32_t>(cur / s);
        r = cur % s;
    }
    big_trim(a);
    return static_cast<uint32_t>(r);
}
static int big_bitlen(const Big& a) {
    for (size_t i = a.size(); i-- > 0;)
        if (a[i]) return static_cast<int>(i) * 32 + (32 - __builtin_clz(a[i]));
    return 0;
}
static uint64_t big_top64(const Big& a, int& shift) {   // a ~= top * 2^shift, top < 2^64
    const int nb = big_bitlen(a);
    shift = nb > 64 ? nb - 64 : 0;
    uint64_t top = 0;
    for (int b = 63; b >= 0; --b) {
        const int bit = shift + b;
        if (bit >= nb) continue;
        if ((a[bit >> 5] >> (bit & 31)) & 1u) top |= (1ull << b);
    }
    return top;
}
static int64_t inv_mod(int64_t a, int64_t p) {   // a^-1 mod p, gcd(a,p) = 1
    int64_t t = 0, nt = 1, r = p, nr = a % p;
    while (nr) { const int64_t q = r / nr; int64_t tmp = t - q * nt; t = nt; nt = tmp; tmp = r - q * nr; r = nr; nr = tmp; }
    return t < 0 ? t + p : t;
}
static int gcd_i(int a, int b) { while (b) { const int t = a % b; a = b; b = t; } return a; }

static std::vector<int> int8_moduli(int N) {
    // greedy pairwise coprime from 256 down (eq. p_list)
    std::vector<int> out;
    for (int c = 256; c >= 2 && static_cast<int>(out.size()) < N; --c) {
        bool ok = true;
        for (int q : out) ok = ok && gcd_i(c, q) == 1;
        if (ok) out.push_back(c);
    }
    return out;
}

static std::vector<int> hybrid_moduli(int N) {
    // squares s^2 > 513 (s <= 33) pairwise coprime, then greedy coprime from 513 down
    std::vector<int> out;
    for (int s = 33; s >= 2 && static_cast<int>(out.size()) < N; --s) {
        const int p = s * s;
        if (p <= 513) break;
        bool ok = true;
        for (int q : out) ok = ok && gcd_i(p, q) == 1;
        if (ok) out.push_back(p);
    }
    for (int c = 513; c >= 2 && static_cast<int>(out.size()) < N; --c) {
        bool ok = true;
        for (int q : out) ok = ok && gcd_i(c, q) == 1;
        if (ok) out.push_back(c);
    }
    return out;
}
static std::vector<int> karatsuba_moduli(int N) {
    // greedy pairwise coprime from 513 down (eq. p_list_karatsuba)
    std::vector<int> out;
    for (int c = 513; c >= 2 && static_cast<int>(out.size()) < N; --c) {
        bool ok = true;
        for (int q : out) ok = ok && gcd_i(c, q) == 1;
        if (ok) out.push_back(c);
    }
    return out;
}
static bool is_square_i(int p) { const int s = static_cast<int>(std::lround(std::sqrt(static_cast<double>(p)))); return s * s == p; }

static float rd32(long double x) {
    float f = static_cast<float>(x);
    if (static_cast<long double>(f) > x) f = std::nextafterf(f, -INFINITY);
    return f;
}
static float ru32(long double x) {
    float f = static_cast<float>(x);
    if (static_cast<long double>(f) < x) f = std::nextafterf(f, INFINITY);
    return f;
}

struct Plan {
    int N = 0, nsq = 0, M = 0, L = 0;
    int family = FAMILY_HYBRID_FP8;
    std::vector<int> p;
    float p_prime = 0, delta = 0;
    double log2P = 0;
    FastExpParams fast{};             // H = RD64((P-1)/2) for fast mode (R15)
    CrtParams crt{};
    DigitParams dig{};
    GemmParams gemm_mod{};            // only .mod[] filled: 3 products per FP8 modulus
    GemmParams gemm_mod_kcat{};       // square moduli with the K-concatenated cross product
    std::vector<uint16_t> pow2tab;    // [N][kPow2Tab]
    uint16_t* d_pow2tab = nullptr;    // device copy (per thread)
    Big P;
    std::vector<Big> w;
};

static Plan build_plan(int N, int family, int sq_order) {
    Plan pl;
    pl.N = N;
    pl.family = family;
    const bool i8 = family == FAMILY_INT8;
    const bool kara = family == FAMILY_KARATSUBA_FP8;   // every modulus takes the Karatsuba digits
    pl.p = i8 ? int8_moduli(N) : kara ? karatsuba_moduli(N) : hybrid_moduli(N);
    if (!i8 && !kara)
        for (int p : pl.p) pl.nsq += is_square_i(p) ? 1 : 0;
    pl.M = i8 ? N : 2 * pl.nsq + 3 * (N - pl.nsq);
    Big P{1};
    for (int p : pl.p) big_mul_small(P, static_cast<uint32_t>(p));
    pl.P = P;
    const int nb = big_bitlen(P);
    // two's complement over L limbs must hold (-1.5 P, 1.5 P): 32 L >= nb + 2; at least
    // 4 limbs (the CRT kernel is instantiated for L = 4..10)
    pl.L = (nb + 2 + 31) / 32;
    if (pl.L < 4) pl.L = 4;
    // P' = RD32((log2(P-1) - 1)/2)
    Big Pm1 = P;
    for (auto& x : Pm1) { if (x--) break; }    // P - 1 (P > 0)
    big_trim(Pm1);
    int sh = 0;
    const uint64_t top = big_top64(Pm1, sh);
    const long double lg = static_cast<long double>(sh) + log2l(static_cast<long double>(top));
    pl.p_prime = rd32((lg - 1.0L) / 2.0L);
    pl.delta = rd32(-1.0L / (2.0L - ldexpl(1.0L, -21)));
    int shP = 0;
    const uint64_t topP = big_top64(P, shP);
    pl.log2P = static_cast<double>(static_cast<long double>(shP) + log2l(static_cast<long double>(topP)));
    {   // H = RD64((P-1)/2).  P is even (1024 | P), so (P-1)/2 = F + 1/2 with F = P/2 - 1:
        // exact as (2F+1) 2^-1 while F < 2^52, else RD64(F) = F truncated to 53 bits.
        Big F = P;
        big_divmod_small(F, 2);
        for (auto& x : F) { if (x--) break; }
        big_trim(F);
        const int fb = big_bitlen(F);
        int sh = 0;
        const uint64_t top = big_top64(F, sh);           // F = top 2^sh (+ lower bits if sh > 0)
        if (fb <= 52) {
            pl.fast.h = 2 * top + 1;
            pl.fast.th = -1;
        } else {
            pl.fast.h = top >> (fb - sh - 53);           // top has fb - sh significant bits
            pl.fast.th = fb - 53;
        }
    }
    // CRT constants
    CrtParams& cp = pl.crt;
    std::memset(&cp, 0, sizeof(cp));
    cp.num_moduli = N;
    for (int l = 0; l < N; ++l) {
        const int p = pl.p[l];
        Big Pp = P;
        big_divmod_small(Pp, static_cast<uint32_t>(p));
        Big tmp = Pp;
        const uint32_t rem = big_divmod_small(tmp, static_cast<uint32_t>(p));
        const int64_t q = inv_mod(rem, p);
        Big w = Pp;
        big_mul_small(w, static_cast<uint32_t>(q));
        pl.w.push_back(w);
        cp.p[l] = p;
        cp.qp32[l] = static_cast<uint32_t>((static_cast<uint64_t>(q) << 32) / static_cast<uint64_t>(p));
        for (int t = 0; t < pl.L && t < static_cast<int>(w.size()); ++t) cp.w[l][t] = w[t];
    }
    for (int t = 0; t < pl.L && t < static_cast<int>(P.size()); ++t) cp.P[t] = P[t];
    {   // np = 2^(32L) - P, halfP = P/2
        uint64_t c = 1;
        for (int t = 0; t < pl.L; ++t) {
            const uint64_t s = static_cast<uint64_t>(~cp.P[t]) + c;
            cp.np[t] = static_cast<uint32_t>(s);
            c = s >> 32;
        }
        for (int t = 0; t < pl.L; ++t) {
            const uint32_t hi = (t + 1 < pl.L) ? cp.P[t + 1] : 0u;
            cp.halfP[t] = (cp.P[t] >> 1) | (hi << 31);
        }
    }
    // digit split and epilogue constants
    DigitParams& dp = pl.dig;
    std::memset(&dp, 0, sizeof(dp));
    dp.num_moduli = N;
    dp.num_planes = pl.M;
    dp.int8 = i8 ? 1 : 0;
    dp.num_squares = pl.nsq;
    dp.even_index = -1;
    {
        int pmin = pl.p[0];
        for (int p : pl.p) pmin = p < pmin ? p : pmin;
        dp.lim1 = std::ldexp(static_cast<double>(pmin), 50);
        dp.lim2 = std::ldexp(static_cast<double>(pmin), 86);
    }
    int plane = 0;
    for (int l = 0; l < N; ++l) {
        const int p = pl.p[l];
        ModDig& md = dp.mod[l];
        md.p_d = p;
        md.pinv_d = 1.0 / p;
        md.p_f = static_cast<float>(p);
        md.pinv_f = 1.0f / static_cast<float>(p);
        md.hp_f = (p % 2 == 0) ? 0.5f / static_cast<float>(p) : 0.0f;
        md.h_f = (p % 2 == 0) ? 0.5f : 0.0f;
        {   // paired residue constants: Q = p_l p_(l+1) <= 1089 * 1024 < 2^21 (exact in FP64)
            const double q2 = (l % 2 == 0 && l + 1 < N) ? static_cast<double>(p) * pl.p[l + 1] : static_cast<double>(p);
            md.q2_d = q2;
            md.q2inv_d = 1.0 / q2;
        }
        if (p % 2 == 0) dp.even_index = l;
        {   // smod(2^(8i), p) in [-floor(p/2), ceil(p/2) - 1]
            int64_t v = 1;
            for (int i = 0; i < 8; ++i) {
                int64_t sv = v % p;
                if (sv >= (p + 1) / 2) sv -= p;
                md.w8[i] = static_cast<float>(sv);
                v = (v * 256) % p;
            }
        }
        md.square = i8 ? 2 : (!kara && is_square_i(p) ? 1 : 0);
        const int s = md.square ? static_cast<int>(std::lround(std::sqrt(static_cast<double>(p)))) : 16;
        md.s_f = static_cast<float>(s);
        md.inv_s_f = 1.0f / static_cast<float>(s);
        md.plane0 = plane;
        ModEpi& me = pl.gemm_mod.mod[l];
        me.p = static_cast<float>(p);
        me.pinv = 1.0f / static_cast<float>(p);
        {
            int64_t w = 65536 % p;
            if (w >= (p + 1) / 2) w -= p;
            me.w16 = static_cast<float>(w);
        }
        me.nprod = 3;
        me.a_plane2 = me.b_plane2 = -1;
        if (i8) {
            // one exact INT8 GEMM per modulus: C'_l = mod(A'_l B'_l, p_l) (eq. CRTmatmul)
            me.coef[0] = 1.0f; me.a_plane[0] = plane; me.b_plane[0] = plane;
            me.nprod = 1;
            plane += 1;
        } else if (md.square) {
            // C'_l = mod(s A1 B2 + s A2 B1 + A2 B2, p)  (eq. 3matmult-notKaratsuba)
            if (sq_order == 1) {
                // A1 B2, A2 B2, A2 B1: consecutive products share B2, then A2, so their
                // operand panels are still in L2 (residue-GEMM DRAM reads 187 -> 178 GB at
                // 16384^3, N = 13); OZ2_SQ_ORDER=0 restores the order of the equation
                me.coef[0] = static_cast<float>(s); me.a_plane[0] = plane + 0; me.b_plane[0] = plane + 1;
                me.coef[1] = 1.0f;                  me.a_plane[1] = plane + 1; me.b_plane[1] = plane + 1;
                me.coef[2] = static_cast<float>(s); me.a_plane[2] = plane + 1; me.b_plane[2] = plane + 0;
            } else {
                me.coef[0] = static_cast<float>(s); me.a_plane[0] = plane + 0; me.b_plane[0] = plane + 1;
                me.coef[1] = static_cast<float>(s); me.a_plane[1] = plane + 1; me.b_plane[1] = plane + 0;
                me.coef[2] = 1.0f;                  me.a_plane[2] = plane + 1; me.b_plane[2] = plane + 1;
            }
            {   // K-concatenated: s (A1 B2 + A2 B1) in ONE accumulator (|sum| <= 2 k 2^8 <=
                // 2^24 for k <= 2^15, exact), then A2 B2 -- 2 drains instead of 3 (the M_N
                // product buffers of P:609, 2 per square modulus)
                ModEpi& mk = pl.gemm_mod_kcat.mod[l];
                mk = me;
                mk.nprod = 2;
                mk.coef[0] = static_cast<float>(s); mk.a_plane[0] = plane + 0; mk.b_plane[0] = plane + 1;
                mk.a_plane2 = plane + 1; mk.b_plane2 = plane + 0;
                mk.coef[1] = 1.0f;                  mk.a_plane[1] = plane + 1; mk.b_plane[1] = plane + 1;
                mk.coef[2] = 0.0f;                  mk.a_plane[2] = mk.b_plane[2] = -1;
            }
            plane += 2;
        } else {
            // A'B' = 256 C1 + C2 + 16 (C3 - C1 - C2)  (eq. C'-Karatsuba)
            me.coef[0] = 240.0f; me.a_plane[0] = plane + 0; me.b_plane[0] = plane + 0;
            me.coef[1] = -15.0f; me.a_plane[1] = plane + 1; me.b_plane[1] = plane + 1;
            me.coef[2] = 16.0f;  me.a_plane[2] = plane + 2; me.b_plane[2] = plane + 2;
            plane += 3;
        }
        if (!md.square || i8) pl.gemm_mod_kcat.mod[l] = me;
    }
    pl.pow2tab.resize(static_cast<size_t>(N) * kPow2Tab);
    for (int l = 0; l < N; ++l) {
        uint32_t v = 1 % pl.p[l];
        for (int e = 0; e < kPow2Tab; ++e) {
            pl.pow2tab[static_cast<size_t>(l) * kPow2Tab + e] = static_cast<uint16_t>(v);
            v = (v * 2) % static_cast<uint32_t>(pl.p[l]);
        }
    }
    return pl;
}

static float f_k_of(int64_t k) {   // reading R5: RU32(1/(1 - k 2^-23))
    return ru32(1.0L / (1.0L - static_cast<long double>(k) * ldexpl(1.0L, -23)));
}

// =================================================================================
// per-thread runtime state

// Resources tied to one device (a host thread that switches devices with cudaSetDevice
// gets a separate set per device; nothing of device A is ever used on device B).
struct DevState {
    int device = -1;
    int num_sms = 0;
    void* own_ws = nullptr;
    size_t own_ws_bytes = 0;
    void* staging = nullptr;
    size_t staging_bytes = 0;
    cudaStream_t copy_stream = nullptr;   // host-pointer calls: D2H of finished C blocks
    cudaEvent_t copy_ev = nullptr;
    int32_t* d_status = nullptr;
    cudaEvent_t ev[8] = {};               // phase timers
    std::map<int, std::unique_ptr<Plan>> plans;   // device copies of the plan tables
    void release() {
        int prev = -1;
        if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); return; }   // runtime gone
        if (prev != device) cudaSetDevice(device);
        cudaDeviceSynchronize();
        if (own_ws) cudaFree(own_ws);
        if (staging) cudaFree(staging);
        if (d_status) cudaFree(d_status);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (copy_ev) cudaEventDestroy(copy_ev);
        for (auto& e : ev) if (e) cudaEventDestroy(e);
        for (auto& kv : plans) if (kv.second->d_pow2tab) cudaFree(kv.second->d_pow2tab);
        plans.clear();
        own_ws = staging = nullptr; own_ws_bytes = staging_bytes = 0;
        d_status = nullptr; copy_stream = nullptr; copy_ev = nullptr;
        for (auto& e : ev) e = nullptr;
        if (prev != device) cudaSetDevice(prev);
        cudaGetLastError();
    }
};

static const int kTuneDefault[OZ2_TUNE_COUNT] = {
    2,    // CTA_GROUP
    1,    // SYNC_LEAD
    4,    // SYNC_CHUNK (4 vs 8: -1.1 % residue GEMM at 16384^3, profiles/round2_knobs.md)
    3,    // L2_PROMO
    0,    // MAX_UNITS
    0,    // TMA_HINT_A
    0,    // TMA_HINT_B
    -1,   // MOD_SPLIT
    -1,   // FUSED_CRT
    1,    // SQ_ORDER
    0,    // CRT_GENERIC
    4,    // HOST_BLOCKS
    -1,   // KCAT: auto = on for k <= 2048 (profiles/round2_kcat_k.md)
    1,    // PRESCALE_2READ (one-read measured 0.1-0.4 ms slower in-step: profiles/round2_prescale_ab.md)
    1000, // EPI_SLEEP (ns)
    0,    // DIGITS_FMA (fewer instructions, but 0.1-0.5 ms slower in-step: profiles/round2_digits_ab.md)
    256,  // TILE_N
};

struct ThreadState {
    cudaStream_t stream = nullptr;
    void* user_ws = nullptr;
    size_t user_ws_bytes = 0;
    int mode = OZ2_MODE_ACCURATE;
    int scheme = OZ2_SCHEME_FP8;          // FAMILY_HYBRID_FP8 / FAMILY_INT8 / FAMILY_KARATSUBA_FP8
    int64_t block_m = 0, block_n = 0;     // forced m/n blocking (0: automatic)
    int64_t last_mb = 0, last_nb = 0;     // blocking used by the last call
    bool timing = false;
    bool timed_last = false;
    int tune[OZ2_TUNE_COUNT];
    std::map<int, std::unique_ptr<DevState>> devs;
    DevState* cur = nullptr;              // state of the current device (ensure_device)
    ThreadState() { std::memcpy(tune, kTuneDefault, sizeof(tune)); }
    ~ThreadState() { release_all(); }
    void release_all() {
        for (auto& kv : devs) kv.second->release();
        devs.clear();
        cur = nullptr;
    }
};
static thread_local ThreadState g_ts;
static inline DevState& D() { return *g_ts.cur; }
static inline int tune(int knob) { return g_ts.tune[knob]; }

static std::mutex g_plan_mutex;
static std::map<int, std::unique_ptr<Plan>> g_host_plans;   // host-only queries

static int plan_key(int N, int family, int sq_order) { return N + 64 * family + 1024 * sq_order; }

static const Plan& host_plan(int N) {   // for the calling thread's scheme
    const int fam = g_ts.scheme;
    const int sq = tune(OZ2_TUNE_SQ_ORDER);
    std::lock_guard<std::mutex> lk(g_plan_mutex);
    auto it = g_host_plans.find(plan_key(N, fam, sq));
    if (it == g_host_plans.end())
        it = g_host_plans.emplace(plan_key(N, fam, sq), std::make_unique<Plan>(build_plan(N, fam, sq))).first;
    return *it->second;
}

static int ensure_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return OZ2_ERR_CUDA;
    if (!g_ts.cur || g_ts.cur->device != dev) {
        auto it = g_ts.devs.find(dev);
        if (it == g_ts.devs.end()) {
            int major = 0, sms = 0;
            if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return OZ2_ERR_CUDA;
            if (major != 10) return OZ2_ERR_NOT_SUPPORTED;
            if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return OZ2_ERR_CUDA;
            auto ds = std::make_unique<DevState>();
            ds->device = dev;
            ds->num_sms = sms;
            it = g_ts.devs.emplace(dev, std::move(ds)).first;
        }
        g_ts.cur = it->second.get();
    }
    if (!D().d_status) {
        if (cudaMalloc(&D().d_status, sizeof(int32_t)) != cudaSuccess) return OZ2_ERR_ALLOC;
        if (cudaMemset(D().d_status, 0, sizeof(int32_t)) != cudaSuccess) return OZ2_ERR_CUDA;
    }
    return OZ2_SUCCESS;
}

static Plan* device_plan(int N, int* err) {
    const int sq = tune(OZ2_TUNE_SQ_ORDER);
    const int key = plan_key(N, g_ts.scheme, sq);
    auto it = D().plans.find(key);
    if (it != D().plans.end()) return it->second.get();
    auto pl = std::make_unique<Plan>(build_plan(N, g_ts.scheme, sq));
    const size_t bytes = pl->pow2tab.size() * sizeof(uint16_t);
    if (cudaMalloc(&pl->d_pow2tab, bytes) != cudaSuccess) { *err = OZ2_ERR_ALLOC; return nullptr; }
    if (cudaMemcpy(pl->d_pow2tab, pl->pow2tab.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
        *err = OZ2_ERR_CUDA;
        return nullptr;
    }
    pl->dig.pow2tab = pl->d_pow2tab;
    Plan* raw = pl.get();
    D().plans.emplace(key, std::move(pl));
    return raw;
}

// =================================================================================
// workspace layout

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
static inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Workspace of one call.  Steps 4-6 may run on (mb x nb) blocks of C (m/n blocking,
// P:629-642): the digit planes then hold one row block of A and one column block of B,
// the residues one block of C, and A-bar / B-bar get their own full-size buffers (steps 1-3
// always run on the whole problem, so the exponents -- and hence C -- are identical to the
// unblocked call).  mb = m and nb = n is the unblocked layout, where A-bar / B-bar live in
// the first digit plane.
struct Layout {
    int64_t m_pad, n_pad, k_pad, mb, nb, mb_pad, nb_pad;
    int M;
    bool blocked;
    size_t maxbits, eprime, rsmax, sumsq, eexp, eloc, prog, abar, bbar, digA, digB, res, total;
};

static Layout make_layout(int64_t m, int64_t n, int64_t k, int N, int M, int64_t mb = 0, int64_t nb = 0) {
    Layout L{};
    L.m_pad = round_up(m, PAD_M);
    L.n_pad = round_up(n, PAD_N);
    L.k_pad = pad_k(k);            // super-chunk layout (oz2_internal.h)
    L.mb = (mb <= 0 || mb >= m) ? m : mb;
    L.nb = (nb <= 0 || nb >= n) ? n : nb;
    L.mb_pad = round_up(L.mb, PAD_M);
    L.nb_pad = round_up(L.nb, PAD_N);
    L.blocked = L.mb < m || L.nb < n;
    L.M = M;
    size_t off = 0;
    const size_t mn = static_cast<size_t>(m + n);
    L.maxbits = off; off = align_up(off + 8 * mn, 256);
    L.eprime = off;  off = align_up(off + 4 * mn, 256);
    L.rsmax = off;   off = align_up(off + 4 * mn, 256);
    L.sumsq = off;   off = align_up(off + 8 * mn, 256);
    L.eexp = off;    off = align_up(off + 4 * mn, 256);
    L.eloc = off;    off = align_up(off + 2 * mn * static_cast<size_t>((k + BK - 1) / BK), 256);   // chunk exponents
    L.prog = off;    off = align_up(off + 8, 1024);           // GEMM progress counter (throttle)
    if (L.blocked) {
        L.abar = off; off = align_up(off + static_cast<size_t>(L.m_pad) * L.k_pad, 1024);
        L.bbar = off; off = align_up(off + static_cast<size_t>(L.n_pad) * L.k_pad, 1024);
    }
    L.digA = off;    off = align_up(off + static_cast<size_t>(M) * L.mb_pad * L.k_pad, 1024);
    L.digB = off;    off = align_up(off + static_cast<size_t>(M) * L.nb_pad * L.k_pad, 1024);
    L.res = off;     off = align_up(off + 2ull * N * static_cast<size_t>(L.mb) * static_cast<size_t>(L.nb), 256);
    L.total = off;
    if (!L.blocked) { L.abar = L.digA; L.bbar = L.digB; }
    return L;
}

// Block sizes for a workspace of `bytes` (multiples of 256, or the full extent): the
// largest column block nb (from n down, halving) for which a row block mb >= min(m, nb)
// fits; B's digits are then split least and A's are recomputed ceil(n/nb) times.
// Returns false if not even 256 x 256 blocks fit.
static bool choose_blocking(int64_t m, int64_t n, int64_t k, int N, int M, size_t bytes,
                            int64_t* mb_out, int64_t* nb_out) {
    if (make_layout(m, n, k, N, M).total <= bytes) { *mb_out = m; *nb_out = n; return true; }
    for (int64_t nb = round_up(n, PAD_N);; nb = round_up(nb / 2, PAD_N)) {
        const int64_t nbe = nb >= n ? n : nb;
        // largest mb (multiple of 256) that fits with this nb
        int64_t lo = 0, hi = round_up(m, PAD_M) / PAD_M;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) / 2;
            const int64_t mbe = mid * PAD_M >= m ? m : mid * PAD_M;
            if (make_layout(m, n, k, N, M, mbe, nbe).total <= bytes) lo = mid; else hi = mid - 1;
        }
        const int64_t mb = lo * PAD_M >= m ? m : lo * PAD_M;
        if (lo > 0 && (mb >= m || mb >= nbe)) { *mb_out = mb; *nb_out = nbe; return true; }
        if (nb <= PAD_N) {
            if (lo > 0) { *mb_out = mb; *nb_out = nbe; return true; }
            return false;
        }
    }
}

// =================================================================================
// TMA descriptors (driver entry point fetched through the runtime; no -lcuda)

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
    static PFN_encodeTiled_t fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_t>(p);
    }
    return fn;
}

// 5-D byte tensor maps, 128B swizzle; the box is 128 bytes of K x box_rows rows, which lands
// in shared memory exactly like the 2-D box of a plain K-major matrix:
//   make_map_planes: digit planes (plane_offset): dims {S bytes, 128 rows,
//                    M planes, KS super-chunks, row blocks}; a 256-row box takes two row
//                    blocks ({128, 128, 1, 1, 2}: the blocks' 128-row slabs are stacked)
//   make_map_plain:  a plain [rows][pitch] matrix with k bytes per row (the raw GEMM):
//                    dims {k, rows, 1, 1, 1}
static bool encode_map5(CUtensorMap* map, const void* base, const cuuint64_t (&dims)[5],
                        const cuuint64_t (&strides)[4], const cuuint32_t (&box)[5]) {
    PFN_encodeTiled_t fn = encode_fn();
    if (!fn) return false;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    // L2 promotion of TMA misses (OZ2_TUNE_L2_PROMO: 0 none, 1 64B, 2 128B, 3 256B)
    const int promo = tune(OZ2_TUNE_L2_PROMO);
    const CUtensorMapL2promotion pr = promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                    : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                 : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<void*>(base), dims, strides,
              const_cast<cuuint32_t*>(box), es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool make_map_planes(CUtensorMap* map, const void* base, int M, uint64_t k_pad, uint64_t rows,
                            uint32_t box_rows) {
    const uint64_t S = static_cast<uint64_t>(super_bytes(static_cast<int64_t>(k_pad))), KS = k_pad / S;
    const uint64_t RB = (rows + kRowBlk - 1) / kRowBlk;
    const cuuint64_t dims[5] = {S, static_cast<cuuint64_t>(kRowBlk), static_cast<cuuint64_t>(M), KS, RB};
    const cuuint64_t strides[4] = {S, S * kRowBlk, S * kRowBlk * M, S * kRowBlk * M * KS};
    const cuuint32_t box[5] = {static_cast<cuuint32_t>(BK), box_rows > static_cast<uint32_t>(kRowBlk) ? kRowBlk : box_rows,
                               1, 1, box_rows > static_cast<uint32_t>(kRowBlk) ? box_rows / kRowBlk : 1};
    return encode_map5(map, base, dims, strides, box);
}
static bool make_map_plain(CUtensorMap* map, const void* base, uint64_t k, uint64_t rows, uint64_t pitch,
                           uint32_t box_rows) {
    const cuuint64_t dims[5] = {k, rows, 1, 1, 1};
    const cuuint64_t strides[4] = {pitch, pitch * rows, pitch * rows, pitch * rows};
    const cuuint32_t box[5] = {static_cast<cuuint32_t>(BK), box_rows, 1, 1, 1};
    return encode_map5(map, base, dims, strides, box);
}

static int super_shift_of(int64_t k_pad) {   // log2(S / BK) of the digit-plane layout
    if (super_bytes(k_pad) != kSuper) return 30;   // one super-chunk per row (S = k_pad)
    int s = 0;
    while ((BK << (s + 1)) <= kSuper) ++s;
    return s;
}

// Epilogue poll interval: the knob, but never more than ~8 ns per k-block of a product (an
// accumulator fills in ~0.45 us per k-block at the capped clock; at small k the epilogue is
// on the critical path and a long sleep would delay the slot hand-back)
static unsigned epi_sleep_ns(int num_k_blocks) {
    const int64_t cap = 8ll * num_k_blocks;
    const int64_t v = tune(OZ2_TUNE_EPI_SLEEP);
    return static_cast<unsigned>(v < cap ? v : cap);
}

static int sync_lead() {   // progress throttle of the residue GEMM (OZ2_TUNE_SYNC_LEAD)
    const int v = tune(OZ2_TUNE_SYNC_LEAD);
    return v < 0 ? 0 : v;
}
// 1: 128x256 CTA tiles; 2: 256x256 CTA-pair tiles; 4: two pairs per cluster sharing A by
// TMA multicast (FP8 kinds only; needs an even number of 256-column tiles, else 2)
// (OZ2_TUNE_CTA_GROUP)
static int cta_group(int64_t n_pad, bool i8) {
    const int v = tune(OZ2_TUNE_CTA_GROUP);
    if (v == 1) return 1;
    if (v == 4 && !i8 && (n_pad / BN) % 2 == 0) return 4;   // the kind::i8 kernels have no multicast variant
    return 2;
}
static int a_box_rows(int cg) { return cg == 4 ? BM / 2 : BM; }
static int b_box_rows(int cg) { return cg == 1 ? BN : BN / 2; }
static int tile_m(int cg) { return cg == 1 ? BM : 2 * BM; }

static void phase_mark(int i) {
    if (!g_ts.timing) return;
    if (!D().ev[i]) cudaEventCreate(&D().ev[i]);
    cudaEventRecord(D().ev[i], g_ts.stream);
}

static int read_timing(float* ms_out, int n) {   // phase times of the last timed call
    if (cudaEventSynchronize(D().ev[6]) != cudaSuccess) return OZ2_ERR_CUDA;
    float v[7];
    for (int i = 0; i < 6; ++i)
        if (cudaEventElapsedTime(&v[i], D().ev[i], D().ev[i + 1]) != cudaSuccess) return OZ2_ERR_CUDA;
    if (cudaEventElapsedTime(&v[6], D().ev[0], D().ev[6]) != cudaSuccess) return OZ2_ERR_CUDA;
    for (int i = 0; i < n && i < 7; ++i) ms_out[i] = v[i];
    return OZ2_SUCCESS;
}

// the CUDA error behind the last OZ2_ERR_CUDA of this thread (oz2_last_cuda_error)
static thread_local int t_last_cuda_error = 0;
static int cuda_fail(cudaError_t e) {
    t_last_cuda_error = static_cast<int>(e);
    return OZ2_ERR_CUDA;
}
#define OZ2_CK(x)                                          \
    do {                                                   \
        const cudaError_t e_ = (x);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_);       \
    } while (0)

// =================================================================================
// the pipeline on device pointers

// Called after the last kernel of column block [j0, j0 + nbj) of C has been enqueued
// (host-pointer calls use it to start that block's device-to-host copy early).
struct BlockHook {
    int64_t nb;                                            // column block size wanted (0: none)
    int (*done)(void* ctx, int64_t j0, int64_t nbj);
    void* ctx;
};

static int run_device(bool a_kmajor, bool b_kmajor, int64_t m, int64_t n, int64_t k, double alpha,
                      const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                      double* C, int64_t ldc, int N, const oz2_options* opt,
                      const BlockHook* hook = nullptr) {
    cudaStream_t st = g_ts.stream;
    int err = OZ2_SUCCESS;
    Plan* pl = device_plan(N, &err);
    if (!pl) return err;
    // debug outputs of whole-problem digit planes / residues need the unblocked layout
    const bool want_full = opt && (opt->digits_a || opt->digits_b || opt->residues);
    int64_t mb = g_ts.block_m, nb = g_ts.block_n;
    if (want_full) mb = nb = 0;
    if (hook && hook->nb > 0 && mb <= 0 && nb <= 0 && !want_full) {
        // column blocks of C for the caller (results are identical to the unblocked call);
        // kept only if that layout fits the caller's workspace
        const Layout Lh = make_layout(m, n, k, N, pl->M, m, hook->nb);
        if (!g_ts.user_ws || Lh.total <= g_ts.user_ws_bytes) { mb = m; nb = hook->nb; }
    }
    uint8_t* ws = nullptr;
    Layout L;
    if (g_ts.user_ws) {
        if (mb <= 0 && nb <= 0 && !want_full) {
            if (!choose_blocking(m, n, k, N, pl->M, g_ts.user_ws_bytes, &mb, &nb)) return OZ2_ERR_WORKSPACE;
        }
        L = make_layout(m, n, k, N, pl->M, mb, nb);
        if (g_ts.user_ws_bytes < L.total) return OZ2_ERR_WORKSPACE;
        ws = static_cast<uint8_t*>(g_ts.user_ws);
    } else {
        L = make_layout(m, n, k, N, pl->M, mb, nb);
        if (D().own_ws_bytes < L.total) {
            if (D().own_ws) { cudaStreamSynchronize(st); cudaFree(D().own_ws); D().own_ws = nullptr; D().own_ws_bytes = 0; }
            if (cudaMalloc(&D().own_ws, L.total) != cudaSuccess) return OZ2_ERR_ALLOC;
            D().own_ws_bytes = L.total;
        }
        ws = static_cast<uint8_t*>(D().own_ws);
    }
    g_ts.last_mb = L.mb;
    g_ts.last_nb = L.nb;
    auto* maxbits = reinterpret_cast<unsigned long long*>(ws + L.maxbits);
    auto* eprime = reinterpret_cast<int32_t*>(ws + L.eprime);
    auto* rsmax = reinterpret_cast<uint32_t*>(ws + L.rsmax);
    auto* sumsq = reinterpret_cast<unsigned long long*>(ws + L.sumsq);
    const bool fast = g_ts.mode == OZ2_MODE_FAST;
    const bool i8 = pl->family == FAMILY_INT8;
    auto* eexp = reinterpret_cast<int32_t*>(ws + L.eexp);
    uint8_t* digA = ws + L.digA;
    uint8_t* digB = ws + L.digB;
    auto* res = reinterpret_cast<int16_t*>(ws + L.res);
    uint8_t* abar = ws + L.abar;     // unblocked: the first digit plane, dead after step 3
    uint8_t* bbar = ws + L.bbar;
    // A-bar / B-bar use the digit-plane layout with `gplanes` planes per super-chunk group:
    // M when they live in plane 0 of the digit buffers, 1 in their own buffers
    const int gplanes = L.blocked ? 1 : pl->M;
    int32_t* e_mu = eexp;
    int32_t* e_nu = eexp + m;

    const bool imported = opt && opt->e_mu_in && opt->e_nu_in;
    int sync_chunk = 1;
    {   // throttle chunks must tile the 512-block K segments: a power of two in [1, 512]
        const int kc = tune(OZ2_TUNE_SYNC_CHUNK);
        while (sync_chunk * 2 <= kc && sync_chunk * 2 <= 512) sync_chunk *= 2;
    }
    g_ts.timed_last = false;
    phase_mark(0);
    OZ2_CK(cudaMemsetAsync(D().d_status, 0, sizeof(int32_t), st));
    if (!imported) {
        // ---- step 1: prescale (eq. def:mu'nu')
        OZ2_CK(cudaMemsetAsync(maxbits, 0, 8 * static_cast<size_t>(m + n), st));
        OZ2_CK(cudaMemsetAsync(rsmax, 0, 4 * static_cast<size_t>(m + n), st));
        if (fast || tune(OZ2_TUNE_PRESCALE_2READ)) {
            // row maxima, then the cast (fast mode: sums of squares instead of A-bar)
            OZ2_CK(launch_rowmax(A, m, k, lda, a_kmajor, maxbits, st));
            OZ2_CK(launch_rowmax(B, n, k, ldb, b_kmajor, maxbits + m, st));
            if (fast) OZ2_CK(cudaMemsetAsync(sumsq, 0, 8 * static_cast<size_t>(m + n), st));
            OZ2_CK(launch_cast(A, m, k, lda, a_kmajor, maxbits, eprime, abar, gplanes, L.m_pad, L.k_pad,
                               D().d_status, fast ? sumsq : nullptr, i8, st));
            OZ2_CK(launch_cast(B, n, k, ldb, b_kmajor, maxbits + m, eprime + m, bbar, gplanes, L.n_pad, L.k_pad,
                               D().d_status, fast ? sumsq + m : nullptr, i8, st));
        } else {
            // one read of A and B: chunk-local casts, then the rescale to the row exponent
            auto* eloc = reinterpret_cast<int16_t*>(ws + L.eloc);
            const int64_t kc = (k + BK - 1) / BK;
            OZ2_CK(launch_cast_local(A, m, k, lda, a_kmajor, maxbits, eloc, abar, gplanes, L.m_pad, L.k_pad, i8, st));
            OZ2_CK(launch_cast_local(B, n, k, ldb, b_kmajor, maxbits + m, eloc + m * kc, bbar, gplanes, L.n_pad,
                                     L.k_pad, i8, st));
            OZ2_CK(launch_rescale(m, k, maxbits, eloc, eprime, D().d_status, abar, gplanes, L.k_pad, i8, st));
            OZ2_CK(launch_rescale(n, k, maxbits + m, eloc + m * kc, eprime + m, D().d_status, bbar, gplanes,
                                  L.k_pad, i8, st));
        }
        if (opt && opt->e_prime_a) OZ2_CK(cudaMemcpyAsync(opt->e_prime_a, eprime, 4 * m, cudaMemcpyDeviceToDevice, st));
        if (opt && opt->e_prime_b) OZ2_CK(cudaMemcpyAsync(opt->e_prime_b, eprime + m, 4 * n, cudaMemcpyDeviceToDevice, st));
        if (opt && opt->abar && k && !fast)
            OZ2_CK(launch_unpack_plane(opt->abar, abar, gplanes, 0, m, k, L.k_pad, st));
        if (opt && opt->bbar && k && !fast)
            OZ2_CK(launch_unpack_plane(opt->bbar, bbar, gplanes, 0, n, k, L.k_pad, st));
        // ---- step 2: bound GEMM C-bar' = A-bar B-bar, row/column maxima
        phase_mark(1);
        if (!fast) {
            const int cg = cta_group(L.n_pad, i8);
            CUtensorMap ta, tb;
            if (!make_map_planes(&ta, abar, gplanes, L.k_pad, L.m_pad, a_box_rows(cg))) return cuda_fail(cudaErrorInvalidValue);
            if (!make_map_planes(&tb, bbar, gplanes, L.k_pad, L.n_pad, b_box_rows(cg))) return cuda_fail(cudaErrorInvalidValue);
            GemmParams gp;
            std::memset(&gp, 0, sizeof(gp));
            gp.m = static_cast<int>(m); gp.n = static_cast<int>(n);
            gp.num_k_blocks = static_cast<int>((k + BK - 1) / BK);   // not the layout's padding
            gp.super_shift = super_shift_of(L.k_pad);
            gp.row_blocked = 1;
            gp.m_tiles = static_cast<int>(L.m_pad / tile_m(cg)); gp.n_tiles = static_cast<int>(L.n_pad / BN);
            gp.rmax = rsmax; gp.smax = rsmax + m;
            // the residue GEMM's progress throttle and lazy epilogue wait apply here too
            gp.sync_lead = sync_lead();
            gp.sync_chunk = sync_chunk;
            gp.epi_sleep_ns = epi_sleep_ns(gp.num_k_blocks);
            gp.max_units = tune(OZ2_TUNE_MAX_UNITS);
            if (gp.sync_lead > 0) {
                gp.progress = reinterpret_cast<unsigned long long*>(ws + L.prog);
                OZ2_CK(cudaMemsetAsync(gp.progress, 0, 8, st));
            }
            OZ2_CK(launch_gemm(i8 ? MODE_BOUND_I8 : MODE_BOUND, cg, 0, ta, tb, gp, D().num_sms, st));
        }
        if (opt && opt->rmax && !fast) OZ2_CK(cudaMemcpyAsync(opt->rmax, rsmax, 4 * m, cudaMemcpyDeviceToDevice, st));
        if (opt && opt->smax && !fast) OZ2_CK(cudaMemcpyAsync(opt->smax, rsmax + m, 4 * n, cudaMemcpyDeviceToDevice, st));
        // ---- step 3: scaling exponents (eq. mu-computation / nu-computation)
        phase_mark(2);
        if (fast) {
            // fast mode: Cauchy-Schwarz over the FP8 / INT8 upper bounds, no bound GEMM (R15, R16)
            OZ2_CK(launch_exps_fast(maxbits, eprime, sumsq, nullptr, m + n, pl->fast, i8 ? 0 : 18, eexp, st));
        } else if (i8) {
            // INT8 accurate mode: exact bound-GEMM row / column maxima (R16)
            OZ2_CK(launch_exps_fast(maxbits, eprime, nullptr, rsmax, m + n, pl->fast, 0, eexp, st));
        } else {
            ExpParams ep{pl->p_prime, pl->delta, f_k_of(k)};
            OZ2_CK(launch_exps(maxbits, eprime, rsmax, m + n, ep, eexp, st));
        }
    } else {
        phase_mark(1);
        phase_mark(2);
        OZ2_CK(cudaMemcpyAsync(e_mu, opt->e_mu_in, 4 * m, cudaMemcpyDeviceToDevice, st));
        OZ2_CK(cudaMemcpyAsync(e_nu, opt->e_nu_in, 4 * n, cudaMemcpyDeviceToDevice, st));
    }
    if (opt && opt->e_mu) OZ2_CK(cudaMemcpyAsync(opt->e_mu, e_mu, 4 * m, cudaMemcpyDeviceToDevice, st));
    if (opt && opt->e_nu) OZ2_CK(cudaMemcpyAsync(opt->e_nu, e_nu, 4 * n, cudaMemcpyDeviceToDevice, st));

    // fuse the CRT into the epilogue for up to 6 limbs (N <= 20) when a product lasts long
    // enough to hide the CRT steps spread over it: measured (profiles/round1_fused_crt_ab.md)
    // FP8 fused wins from k = 16384 on (+1-2 %) and loses 20 % at k = 8192; INT8 (one
    // product per modulus, so 3x the CRT work per product) loses 23 % at k = 16384.
    // OZ2_TUNE_FUSED_CRT: -1 auto (default), 0 never, 1 whenever L <= 6 and k >= 8192.
    const int fuse_env = tune(OZ2_TUNE_FUSED_CRT);
    const bool fuse_auto = i8 ? k >= 49152 : k >= 16384;
    const int fused = (pl->L <= 6 && k >= 8192 && (fuse_env > 0 || (fuse_env < 0 && fuse_auto))) ? pl->L : 0;
    // ---- steps 4-6 on blocks of C (one block when unblocked)
    phase_mark(3);
    if (L.blocked) phase_mark(4);     // blocked: the whole block loop counts as "residue GEMM"
    for (int64_t j0 = 0; j0 < n; j0 += L.nb) {
        const int64_t nbj = std::min(L.nb, n - j0), nbj_pad = round_up(nbj, PAD_N);
        const double* Bj = b_kmajor ? B + j0 * ldb : B + j0;
        // ---- step 4: integers, residues, FP8 digits
        // row maxima of step 1 (not computed when the exponents are imported)
        const unsigned long long* mx = (imported || !tune(OZ2_TUNE_DIGITS_FMA)) ? nullptr : maxbits;
        OZ2_CK(launch_digits(Bj, nbj, k, ldb, b_kmajor, e_nu + j0, mx ? mx + m + j0 : nullptr, pl->dig, digB,
                             nbj_pad, L.k_pad, st));
        for (int64_t i0 = 0; i0 < m; i0 += L.mb) {
            const int64_t mbi = std::min(L.mb, m - i0), mbi_pad = round_up(mbi, PAD_M);
            const double* Ai = a_kmajor ? A + i0 * lda : A + i0;
            if (j0 == 0 || L.mb < m)      // one row block: A's digits survive across column blocks
                OZ2_CK(launch_digits(Ai, mbi, k, lda, a_kmajor, e_mu + i0, mx ? mx + i0 : nullptr, pl->dig, digA,
                                     mbi_pad, L.k_pad, st));
            if (!L.blocked) {
                if (opt && opt->digits_a && k)
                    for (int x = 0; x < pl->M; ++x)
                        OZ2_CK(launch_unpack_plane(opt->digits_a + static_cast<size_t>(x) * m * k, digA, pl->M, x,
                                                   m, k, L.k_pad, st));
                if (opt && opt->digits_b && k)
                    for (int x = 0; x < pl->M; ++x)
                        OZ2_CK(launch_unpack_plane(opt->digits_b + static_cast<size_t>(x) * n * k, digB, pl->M, x,
                                                   n, k, L.k_pad, st));
                phase_mark(4);
            }
            // ---- step 5: 3N exact FP8 GEMMs with the modular epilogue
            const int cg = cta_group(nbj_pad, i8);
            CUtensorMap ta, tb;
            if (!make_map_planes(&ta, digA, pl->M, L.k_pad, mbi_pad, a_box_rows(cg))) return cuda_fail(cudaErrorInvalidValue);
            if (!make_map_planes(&tb, digB, pl->M, L.k_pad, nbj_pad, b_box_rows(cg))) return cuda_fail(cudaErrorInvalidValue);
            // square moduli: A1 B2 + A2 B1 K-concatenated in one accumulator when the sum
            // stays in the FP32 exactness window (k <= 2^15; OZ2_TUNE_KCAT)
            // (auto: k <= 2048, where each product's MMAs are shorter than its accumulator drain
            // and 33 drains per tile instead of 39 pay: +14 % at 16384^2 x 1024, +7.5 % at 2048;
            // -1 to -2 % from k = 4096 on, profiles/round2_kcat_k.md)
            const int kcat_knob = tune(OZ2_TUNE_KCAT);
            const bool kcat = (kcat_knob > 0 || (kcat_knob < 0 && k <= 2048)) && !i8 && pl->nsq > 0 && k <= kMaxK / 2;
            GemmParams gp = kcat ? pl->gemm_mod_kcat : pl->gemm_mod;
            gp.prods_per_tile = 0;
            for (int l = 0; l < N; ++l) gp.prods_per_tile += gp.mod[l].nprod;
            gp.m = static_cast<int>(mbi); gp.n = static_cast<int>(nbj);
            gp.num_k_blocks = static_cast<int>((k + BK - 1) / BK);   // not the layout's padding
            gp.super_shift = super_shift_of(L.k_pad);
            gp.row_blocked = 1;
            gp.kseg_blocks = kMaxK / BK;                                  // 2^16 per segment
            gp.num_kseg = (gp.num_k_blocks + gp.kseg_blocks - 1) / gp.kseg_blocks;
            // OZ2_TUNE_TILE_N = 512: 256 x 512 CTA-pair tiles (FP8 schemes, CTA pairs)
            const int tile_n = (tune(OZ2_TUNE_TILE_N) == 512 && cg == 2 && !i8) ? 512 : 256;
            gp.m_tiles = static_cast<int>(mbi_pad / tile_m(cg));
            gp.n_tiles = static_cast<int>((nbj_pad + tile_n - 1) / tile_n);
            gp.num_moduli = N;
            {   // work items (OZ2_TUNE_MOD_SPLIT: -1 auto, 0 tile-major, 1 all (tile, modulus),
                // 2 hybrid): few tiles (< 8 per persistent unit) -> all split; otherwise
                // tile-major, with the last partial wave split over all units (hybrid) when
                // it would leave more than 0.5 % of the unit-time idle
                const int64_t tiles = static_cast<int64_t>(gp.m_tiles) * gp.n_tiles / (cg == 4 ? 2 : 1);
                const int64_t units = std::max<int64_t>(1, D().num_sms / (cg == 1 ? 1 : cg == 4 ? 4 : 2));
                const int64_t full = tiles / units * units;
                const int64_t waves = (tiles + units - 1) / units;
                const bool ragged = full < tiles && static_cast<double>(waves * units - tiles) > 0.005 * waves * units;
                int ms = tune(OZ2_TUNE_MOD_SPLIT);
                // hybrid also with the fused CRT (round 2): the head tiles keep their fused CRT,
                // the split tail's tiles get theirs from k_crt_tiles after the GEMM
                if (ms < 0) ms = tiles < 8 * units ? 1 : (ragged ? 2 : 0);
                gp.tail_head = static_cast<int>(ms == 1 ? 0 : ms == 2 ? full : tiles);
            }
            // the fused CRT needs every modulus of a tile in one item: it covers the tile-major
            // head items [0, tail_head); the split tail's CRT runs in k_crt_tiles below
            const int n_tiles_blk = gp.m_tiles * gp.n_tiles / (cg == 4 ? 2 : 1);
            const int fused_blk = gp.tail_head == 0 ? 0 : fused;
            gp.residues = res;
            gp.sync_lead = sync_lead();
            gp.sync_chunk = sync_chunk;
            gp.epi_sleep_ns = epi_sleep_ns(gp.num_k_blocks);
            gp.max_units = tune(OZ2_TUNE_MAX_UNITS);
            {   // OZ2_TUNE_TMA_HINT_A / _B: 0 evict-normal (default), 1 evict-last, 2 evict-first
                auto hint = [](int v) -> unsigned long long {
                    return v == 1 ? 0x14F0000000000000ull : v == 2 ? 0x12F0000000000000ull : 0x1000000000000000ull;
                };
                gp.hint_a = hint(tune(OZ2_TUNE_TMA_HINT_A));
                gp.hint_b = hint(tune(OZ2_TUNE_TMA_HINT_B));
            }
            if (gp.sync_lead > 0) {
                gp.progress = reinterpret_cast<unsigned long long*>(ws + L.prog);
                OZ2_CK(cudaMemsetAsync(gp.progress, 0, 8, st));
            }
            double* Cij = C + i0 + j0 * ldc;
            if (fused_blk) {
                gp.crt = pl->crt;
                gp.e_mu = e_mu + i0; gp.e_nu = e_nu + j0;
                gp.alpha = alpha; gp.beta = beta;
                gp.C = Cij; gp.ldc = ldc;
            }
            OZ2_CK(launch_gemm(i8 ? MODE_RESIDUE_I8 : MODE_RESIDUE, cg, fused_blk, ta, tb, gp, D().num_sms, st, tile_n));
            if (!L.blocked) {
                if (opt && opt->residues)   // stored as u_l in [0, p_l): symmetric C'_l for the caller
                    OZ2_CK(launch_res_symmetric(opt->residues, res, m * n, pl->crt, st));
                phase_mark(5);
            }
            // ---- step 6: CRT + inverse scaling (eqs. CRT_finalreduction, inversescaling)
            if (!fused_blk)
                OZ2_CK(launch_crt(pl->L, res, mbi, nbj, pl->crt, e_mu + i0, e_nu + j0, alpha, beta, Cij, ldc,
                                  tune(OZ2_TUNE_CRT_GENERIC) != 0, st));
            else if (gp.tail_head < n_tiles_blk)
                OZ2_CK(launch_crt_tiles(pl->L, res, mbi, nbj, pl->crt, e_mu + i0, e_nu + j0, alpha, beta, Cij, ldc,
                                        gp.tail_head, n_tiles_blk - gp.tail_head, 16 / (cg == 1 ? 1 : 2), gp.m_tiles,
                                        gp.n_tiles / (cg == 4 ? 2 : 1), tile_m(cg), tile_n * (cg == 4 ? 2 : 1), st));
        }
        if (hook && hook->done) {
            const int hr = hook->done(hook->ctx, j0, nbj);
            if (hr) return hr;
        }
    }
    if (L.blocked) phase_mark(5);
    phase_mark(6);
    g_ts.timed_last = g_ts.timing;
    return OZ2_SUCCESS;
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static bool is_pinned_host(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeHost;
}

static bool trans_ok(char t) {
    return t == 'N' || t == 'n' || t == 'T' || t == 't' || t == 'C' || t == 'c';
}
static bool is_n(char t) { return t == 'N' || t == 'n'; }

static int dgemm_call(char transa, char transb, int64_t m, int64_t n, int64_t k, double alpha,
                      const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                      int64_t ldc, int N, const oz2_options* opt);

// Per-call settings of oz2_options (mode, scheme, timing) applied for the duration of one
// call and restored afterwards (the thread's settings are the defaults).
int dgemm_impl(char transa, char transb, int64_t m, int64_t n, int64_t k, double alpha,
               const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
               int64_t ldc, int N, const oz2_options* opt) {
    if (opt) {
        for (int i = 0; i < 4; ++i) if (opt->reserved[i]) return -15;
        if (opt->set_mode && opt->mode != OZ2_MODE_ACCURATE && opt->mode != OZ2_MODE_FAST) return -15;
        if (opt->set_scheme && opt->scheme != OZ2_SCHEME_FP8 && opt->scheme != OZ2_SCHEME_INT8 &&
            opt->scheme != OZ2_SCHEME_FP8_KARATSUBA) return -15;
    }
    const int mode0 = g_ts.mode, scheme0 = g_ts.scheme;
    const bool timing0 = g_ts.timing;
    if (opt && opt->set_mode) g_ts.mode = opt->mode;
    if (opt && opt->set_scheme) g_ts.scheme = opt->scheme;
    if (opt && opt->timing_ms) g_ts.timing = true;
    int rc = dgemm_call(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, N, opt);
    if (rc == OZ2_SUCCESS && opt && opt->timing_ms) {
        if (g_ts.timed_last) rc = read_timing(opt->timing_ms, 7);
        else for (int i = 0; i < 7; ++i) opt->timing_ms[i] = 0.0f;   // quick return: nothing ran
    }
    g_ts.mode = mode0;
    g_ts.scheme = scheme0;
    g_ts.timing = timing0;
    return rc;
}

static int dgemm_call(char transa, char transb, int64_t m, int64_t n, int64_t k, double alpha,
                      const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                      int64_t ldc, int N, const oz2_options* opt) {
    // BLAS argument checks (xerbla order)
    if (!trans_ok(transa)) return -1;
    if (!trans_ok(transb)) return -2;
    if (m < 0) return -3;
    if (n < 0) return -4;
    if (k < 0) return -5;
    const int64_t rowsA = is_n(transa) ? m : k;
    const int64_t rowsB = is_n(transb) ? k : n;
    if (lda < (rowsA > 1 ? rowsA : 1)) return -8;
    if (ldb < (rowsB > 1 ? rowsB : 1)) return -10;
    if (ldc < (m > 1 ? m : 1)) return -13;
    if (N < 2 || N > kMaxModuli) return -14;
    g_ts.timed_last = false;
    if (m == 0 || n == 0) return OZ2_SUCCESS;
    int e = ensure_device();
    if (e) return e;
    if (k > kMaxKTotal) return OZ2_ERR_NOT_SUPPORTED;      // f_k = 1/(1 - k 2^-23) needs k << 2^23
    if (g_ts.scheme == OZ2_SCHEME_INT8 && k > kMaxK) return OZ2_ERR_NOT_SUPPORTED;   // exact S32 bound (R16)
    if (m > kMaxRows || n > kMaxRows) return OZ2_ERR_NOT_SUPPORTED;   // conversion-kernel grids
    cudaStream_t st = g_ts.stream;
    const bool quick = (alpha == 0.0 || k == 0);
    const bool dev = is_device_ptr(C);
    if (!quick && (dev != is_device_ptr(A) || dev != is_device_ptr(B))) return OZ2_ERR_NOT_SUPPORTED;
    if (dev) {
        if (quick) { OZ2_CK(launch_scale(C, m, n, ldc, beta, st)); return OZ2_SUCCESS; }
        return run_device(!is_n(transa), is_n(transb), m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, N, opt);
    }
    // host buffers: stage through device memory, run, copy back, synchronise
    const int64_t colsA = is_n(transa) ? k : m;
    const int64_t colsB = is_n(transb) ? n : k;
    const size_t bA = align_up(8ull * rowsA * colsA, 256), bB = align_up(8ull * rowsB * colsB, 256);
    const size_t bC = align_up(8ull * m * n, 256);
    const size_t need = bA + bB + bC;
    if (D().staging_bytes < need) {
        if (D().staging) { cudaStreamSynchronize(st); cudaFree(D().staging); D().staging = nullptr; D().staging_bytes = 0; }
        if (cudaMalloc(&D().staging, need) != cudaSuccess) return OZ2_ERR_ALLOC;
        D().staging_bytes = need;
    }
    double* dA = static_cast<double*>(D().staging);
    double* dB = reinterpret_cast<double*>(static_cast<uint8_t*>(D().staging) + bA);
    double* dC = reinterpret_cast<double*>(static_cast<uint8_t*>(D().staging) + bA + bB);
    if (!quick) {
        OZ2_CK(cudaMemcpy2DAsync(dA, 8 * rowsA, A, 8 * lda, 8 * rowsA, colsA, cudaMemcpyHostToDevice, st));
        OZ2_CK(cudaMemcpy2DAsync(dB, 8 * rowsB, B, 8 * ldb, 8 * rowsB, colsB, cudaMemcpyHostToDevice, st));
    }
    if (beta != 0.0) OZ2_CK(cudaMemcpy2DAsync(dC, 8 * m, C, 8 * ldc, 8 * m, n, cudaMemcpyHostToDevice, st));
    int rc = OZ2_SUCCESS;
    if (quick) {
        rc = launch_scale(dC, m, n, m, beta, st) == cudaSuccess ? OZ2_SUCCESS : OZ2_ERR_CUDA;
        if (rc) return rc;
        OZ2_CK(cudaMemcpy2DAsync(C, 8 * ldc, dC, 8 * m, 8 * m, n, cudaMemcpyDeviceToHost, st));
        OZ2_CK(cudaStreamSynchronize(st));
        return OZ2_SUCCESS;
    }
    // C goes back in column blocks: block j's device-to-host copy (on a second stream)
    // overlaps the GEMMs of blocks j+1.. (OZ2_HOST_BLOCKS blocks, default 4; 1 = off)
    if (!D().copy_stream) {
        OZ2_CK(cudaStreamCreateWithFlags(&D().copy_stream, cudaStreamNonBlocking));
        OZ2_CK(cudaEventCreateWithFlags(&D().copy_ev, cudaEventDisableTiming));
    }
    struct Ctx { double* C; int64_t ldc; const double* dC; int64_t m; } ctx{C, ldc, dC, m};
    BlockHook hook{};
    // (a copy into pageable memory is synchronous with the host, which would serialise
    // the blocks: only pinned C is copied in blocks)
    const int nblk = tune(OZ2_TUNE_HOST_BLOCKS);
    if (nblk > 1 && n >= 2 * PAD_N * nblk && is_pinned_host(C)) hook.nb = round_up((n + nblk - 1) / nblk, PAD_N);
    hook.ctx = &ctx;
    hook.done = [](void* c, int64_t j0, int64_t nbj) -> int {
        const Ctx& x = *static_cast<const Ctx*>(c);
        if (cudaEventRecord(D().copy_ev, g_ts.stream) != cudaSuccess) return OZ2_ERR_CUDA;
        if (cudaStreamWaitEvent(D().copy_stream, D().copy_ev, 0) != cudaSuccess) return OZ2_ERR_CUDA;
        if (cudaMemcpy2DAsync(x.C + j0 * x.ldc, 8 * x.ldc, x.dC + j0 * x.m, 8 * x.m, 8 * x.m, nbj,
                              cudaMemcpyDeviceToHost, D().copy_stream) != cudaSuccess)
            return OZ2_ERR_CUDA;
        return OZ2_SUCCESS;
    };
    rc = run_device(!is_n(transa), is_n(transb), m, n, k, alpha, dA, rowsA, dB, rowsB, beta, dC, m, N, opt, &hook);
    const cudaError_t e1 = cudaStreamSynchronize(st);
    const cudaError_t e2 = cudaStreamSynchronize(D().copy_stream);
    if (rc) return rc;
    if (e1 != cudaSuccess || e2 != cudaSuccess) return OZ2_ERR_CUDA;
    return OZ2_SUCCESS;
}

}  // namespace oz2

using namespace oz2;

// =================================================================================
// C ABI

extern "C" {

int oz2_dgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, double alpha,
              const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
              int64_t ldc, int num_moduli) {
    return dgemm_impl(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, num_moduli, nullptr);
}

int oz2_dgemm_ex(char transa, char transb, int64_t m, int64_t n, int64_t k, double alpha,
                 const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                 int64_t ldc, int num_moduli, const oz2_options* opt) {
    return dgemm_impl(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, num_moduli, opt);
}

int oz2_set_stream(void* stream) {
    g_ts.stream = static_cast<cudaStream_t>(stream);
    return OZ2_SUCCESS;
}

size_t oz2_workspace_size(char transa, char transb, int64_t m, int64_t n, int64_t k, int num_moduli) {
    if (!trans_ok(transa) || !trans_ok(transb) || m < 0 || n < 0 || k < 0) return 0;
    if (num_moduli < 2 || num_moduli > kMaxModuli) return 0;
    const Plan& pl = host_plan(num_moduli);
    return make_layout(m, n, k, num_moduli, pl.M).total;
}

int oz2_set_mode(int mode) {
    if (mode != OZ2_MODE_ACCURATE && mode != OZ2_MODE_FAST) return -1;
    g_ts.mode = mode;
    return OZ2_SUCCESS;
}

int oz2_get_mode(void) { return g_ts.mode; }

int oz2_set_scheme(int scheme) {
    if (scheme != OZ2_SCHEME_FP8 && scheme != OZ2_SCHEME_INT8 && scheme != OZ2_SCHEME_FP8_KARATSUBA) return -1;
    g_ts.scheme = scheme;
    return OZ2_SUCCESS;
}

int oz2_get_scheme(void) { return g_ts.scheme; }

int oz2_set_blocking(int64_t mb, int64_t nb) {
    if (mb < 0) return -1;
    if (nb < 0) return -2;
    if ((mb % PAD_M) != 0) return -1;
    if ((nb % PAD_N) != 0) return -2;
    g_ts.block_m = mb;
    g_ts.block_n = nb;
    return OZ2_SUCCESS;
}

int oz2_get_blocking(int64_t* mb, int64_t* nb) {
    if (!mb) return -1;
    if (!nb) return -2;
    *mb = g_ts.last_mb;
    *nb = g_ts.last_nb;
    return OZ2_SUCCESS;
}

size_t oz2_workspace_size_blocked(int64_t m, int64_t n, int64_t k, int num_moduli, int64_t mb, int64_t nb) {
    if (m < 0 || n < 0 || k < 0 || mb < 0 || nb < 0) return 0;
    if (num_moduli < 2 || num_moduli > kMaxModuli) return 0;
    const Plan& pl = host_plan(num_moduli);
    return make_layout(m, n, k, num_moduli, pl.M, mb, nb).total;
}

int oz2_plan_blocking(int64_t m, int64_t n, int64_t k, int num_moduli, size_t bytes, int64_t* mb,
                      int64_t* nb) {
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (k < 0) return -3;
    if (num_moduli < 2 || num_moduli > kMaxModuli) return -4;
    if (!mb) return -6;
    if (!nb) return -7;
    const Plan& pl = host_plan(num_moduli);
    return choose_blocking(m, n, k, num_moduli, pl.M, bytes, mb, nb) ? OZ2_SUCCESS : OZ2_ERR_WORKSPACE;
}

int oz2_set_workspace(void* ptr, size_t bytes) {
    g_ts.user_ws = ptr;
    g_ts.user_ws_bytes = ptr ? bytes : 0;
    return OZ2_SUCCESS;
}

int oz2_get_status(int32_t* status) {
    if (!status) return -1;
    int e = ensure_device();
    if (e) return e;
    int32_t h = 0;
    OZ2_CK(cudaStreamSynchronize(g_ts.stream));
    OZ2_CK(cudaMemcpy(&h, D().d_status, sizeof(h), cudaMemcpyDeviceToHost));
    OZ2_CK(cudaMemset(D().d_status, 0, sizeof(int32_t)));
    *status = h ? OZ2_ERR_NONFINITE : OZ2_SUCCESS;
    return OZ2_SUCCESS;
}

int oz2_set_timing(int enable) {
    g_ts.timing = enable != 0;
    return OZ2_SUCCESS;
}

int oz2_get_timing(float* ms_out, int n) {
    if (!ms_out) return -1;
    if (!g_ts.timed_last || !g_ts.cur) return OZ2_ERR_NOT_SUPPORTED;
    return read_timing(ms_out, n);
}


int oz2_last_cuda_error(char* name_out, int cap) {
    const int e = t_last_cuda_error;
    if (name_out && cap > 0) {
        const char* nm = cudaGetErrorName(static_cast<cudaError_t>(e));
        int i = 0;
        for (; nm && nm[i] && i < cap - 1; ++i) name_out[i] = nm[i];
        name_out[i] = 0;
    }
    return e;
}

int oz2_finalize(void) {
    if (g_ts.stream) cudaStreamSynchronize(g_ts.stream);
    g_ts.release_all();
    return OZ2_SUCCESS;
}

int oz2_set_tuning(int knob, int value) {
    if (knob < 0 || knob >= OZ2_TUNE_COUNT) return -1;
    bool ok = true;
    switch (knob) {
        case OZ2_TUNE_CTA_GROUP: ok = value == 1 || value == 2 || value == 4; break;
        case OZ2_TUNE_SYNC_LEAD: ok = value >= 0 && value <= 1 << 20; break;
        case OZ2_TUNE_SYNC_CHUNK: ok = value >= 1 && value <= 512; break;
        case OZ2_TUNE_L2_PROMO: ok = value >= 0 && value <= 3; break;
        case OZ2_TUNE_MAX_UNITS: ok = value >= 0; break;
        case OZ2_TUNE_TMA_HINT_A:
        case OZ2_TUNE_TMA_HINT_B: ok = value >= 0 && value <= 2; break;
        case OZ2_TUNE_MOD_SPLIT: ok = value >= -1 && value <= 2; break;
        case OZ2_TUNE_FUSED_CRT: ok = value >= -1 && value <= 1; break;
        case OZ2_TUNE_SQ_ORDER:
        case OZ2_TUNE_CRT_GENERIC:
        case OZ2_TUNE_KCAT: ok = value >= -1 && value <= 1; break;
        case OZ2_TUNE_PRESCALE_2READ: ok = value == 0 || value == 1; break;
        case OZ2_TUNE_HOST_BLOCKS: ok = value >= 1 && value <= 64; break;
        case OZ2_TUNE_EPI_SLEEP: ok = value >= 0 && value <= 100000; break;
        case OZ2_TUNE_DIGITS_FMA: ok = value == 0 || value == 1; break;
        case OZ2_TUNE_TILE_N: ok = value == 256 || value == 512; break;
        default: break;
    }
    if (!ok) return -2;
    g_ts.tune[knob] = value;
    return OZ2_SUCCESS;
}

int oz2_get_tuning(int knob, int* value) {
    if (knob < 0 || knob >= OZ2_TUNE_COUNT) return -1;
    if (!value) return -2;
    *value = g_ts.tune[knob];
    return OZ2_SUCCESS;
}

void oz2_reset_tuning(void) { std::memcpy(g_ts.tune, kTuneDefault, sizeof(g_ts.tune)); }

int oz2_moduli(int num_moduli, int32_t* p_out) {
    if (num_moduli < 2 || num_moduli > kMaxModuli) return -1;
    if (!p_out) return -2;
    const Plan& pl = host_plan(num_moduli);
    for (int l = 0; l < num_moduli; ++l) p_out[l] = pl.p[l];
    return OZ2_SUCCESS;
}

int oz2_plan_query(int num_moduli, int64_t k, oz2_plan_info* out) {
    if (num_moduli < 2 || num_moduli > kMaxModuli) return -1;
    if (k < 0) return -2;
    if (!out) return -3;
    const Plan& pl = host_plan(num_moduli);
    std::memset(out, 0, sizeof(*out));
    out->num_moduli = num_moduli;
    out->num_planes = pl.M;
    out->num_limbs = pl.L;
    out->num_squares = pl.nsq;
    out->p_prime = pl.p_prime;
    out->delta = pl.delta;
    out->f_k = f_k_of(k);
    out->log2_P = pl.log2P;
    out->fast_H = std::ldexp(static_cast<double>(pl.fast.h), pl.fast.th);
    for (int t = 0; t < pl.L && t < 12; ++t) out->P_limbs[t] = pl.crt.P[t];
    for (int l = 0; l < num_moduli; ++l)
        for (int t = 0; t < pl.L && t < 12; ++t) out->w_limbs[l][t] = pl.crt.w[l][t];
    return OZ2_SUCCESS;
}

const char* oz2_version(void) { return "oz2 0.1.0 sm_100a"; }

static int gemm_raw(int mode, const uint8_t* a, const uint8_t* b, float* C32, int64_t m, int64_t n, int64_t k,
                    uint32_t* rmax = nullptr, uint32_t* smax = nullptr);

int oz2_fp8_gemm_bound(const uint8_t* a, const uint8_t* b, uint32_t* rmax, uint32_t* smax, int64_t m, int64_t n,
                       int64_t k) {
    if (!rmax && m > 0) return -3;
    if (!smax && n > 0) return -4;
    return gemm_raw(MODE_BOUND, a, b, nullptr, m, n, k, rmax, smax);
}

int oz2_fp8_gemm_raw(const uint8_t* a, const uint8_t* b, float* C32, int64_t m, int64_t n, int64_t k) {
    return gemm_raw(MODE_RAW, a, b, C32, m, n, k);
}

int oz2_int8_gemm_raw(const int8_t* a, const int8_t* b, int32_t* C32, int64_t m, int64_t n, int64_t k) {
    return gemm_raw(MODE_RAW_I8, reinterpret_cast<const uint8_t*>(a), reinterpret_cast<const uint8_t*>(b),
                    reinterpret_cast<float*>(C32), m, n, k);
}

static int gemm_raw(int mode, const uint8_t* a, const uint8_t* b, float* C32, int64_t m, int64_t n, int64_t k,
                    uint32_t* rmax, uint32_t* smax) {
    if (m < 0) return -4;
    if (n < 0) return -5;
    if (k < 0 || (k % 16) != 0) return -6;
    if (m == 0 || n == 0) return OZ2_SUCCESS;
    int e = ensure_device();
    if (e) return e;
    if (k == 0) {
        if (C32) OZ2_CK(cudaMemsetAsync(C32, 0, 4ull * m * n, g_ts.stream));
        return OZ2_SUCCESS;
    }
    if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15u) return OZ2_ERR_NOT_SUPPORTED;
    const int cg = cta_group(((n + BN - 1) / BN) * BN, mode == MODE_RAW_I8);
    CUtensorMap ta, tb;
    if (!make_map_plain(&ta, a, k, m, k, a_box_rows(cg))) return cuda_fail(cudaErrorInvalidValue);
    if (!make_map_plain(&tb, b, k, n, k, b_box_rows(cg))) return cuda_fail(cudaErrorInvalidValue);
    GemmParams gp;
    std::memset(&gp, 0, sizeof(gp));
    gp.m = static_cast<int>(m); gp.n = static_cast<int>(n);
    gp.num_k_blocks = static_cast<int>((k + BK - 1) / BK);
    gp.m_tiles = static_cast<int>((m + tile_m(cg) - 1) / tile_m(cg)); gp.n_tiles = static_cast<int>((n + BN - 1) / BN);
    gp.c32 = C32;
    gp.rmax = rmax;
    gp.smax = smax;
    gp.super_shift = 30;           // plain [rows][k] operands
    OZ2_CK(launch_gemm(mode, cg, 0, ta, tb, gp, D().num_sms, g_ts.stream));
    return OZ2_SUCCESS;
}

}  // extern "C"
