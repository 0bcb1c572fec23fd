// gemm_kernel.cu -- the FP8 (E4M3 x E4M3 -> FP32) GEMMs of the FP8 Ozaki-II scheme on
// 5th-generation tensor cores (tcgen05.mma kind::f8f6f4), persistent, one CTA per SM.
//
// CG = 1: one CTA computes a 128 x 256 tile (UMMA M=128, N=256).
// CG = 2: a cluster of two CTAs on one TPC computes a 256 x 256 tile with
//         tcgen05.mma.cta_group::2 (UMMA M=256, N=256) issued by the leader CTA: each
//         CTA stages its own 128 rows of A and half (128 rows) of B^T, the tensor core
//         reads both halves, and each CTA's TMEM receives its 128 rows x 256 columns.
//         Per SM this halves the B bytes moved from L2 and read from shared memory.
//
// Roles (320 threads per CTA):
//   warp 0      TMA producer (K-major operand tiles, 128-byte swizzle, NSTAGE-deep ring)
//   warp 1      TMEM allocator + single-thread MMA issuer (leader CTA only for CG = 2):
//               4 x K=32 MMAs per 128-byte K stage into one of two 256-column FP32
//               accumulators in TMEM (double buffer: the epilogue of product g overlaps
//               the MMAs of product g+1)
//   warps 2..9  epilogue: tcgen05.ld 32 lanes x 32 columns; warp w reads TMEM lane
//               quadrant w % 4 and one 128-column half of the tile
//
// Modes:
//   MODE_RESIDUE  for every tile and every modulus l the three exact products of
//                 P:292-299 (square p = s^2: A1 B2, A2 B1, A2 B2 with weights s, s, 1)
//                 or eq. C'-Karatsuba P:241-246 (non-square: A^x B^x, x = 1..3 with
//                 weights 256-16, 1-16, 16) run back to back; the epilogue reduces
//                 each FP32 accumulator mod p (exact: entries are integers <= 2^24,
//                 eq. error-free-FP8-matmult), accumulates the weighted partial in
//                 registers (binary16 pairs, exact below 2048) and after the third
//                 product stores C'_l mod p in [0, p) as 16 bits [l][j][i] (work
//                 items: a tile with all moduli, or one (tile, modulus) pair when
//                 mod_split); with FL > 0 the CRT of the previous tile is spread over
//                 the epilogues (crt_common.cuh).  The FP32 products never leave TMEM.
//   MODE_BOUND    C-bar' = A-bar B-bar; the epilogue keeps only the row and
//                 column maxima (atomicMax on non-negative float bits).
//   MODE_RAW      diagnostic: writes the FP32 accumulator.
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include "oz2_internal.h"
#include "oz2_ptx.cuh"
#include "crt_common.cuh"

namespace oz2 {

// W = 2 (CG = 2, residue mode only): a 256 x 512 tile per CTA pair -- two N = 256 MMAs per
// K step share the staged A tile (25 % fewer operand bytes per MAC moved L2 -> SM), the two
// 256-column accumulators are the L and R halves of the tile (no double buffer: the next
// product's L half starts as soon as L is drained, see the MMA issuer), and each epilogue
// thread keeps the partial residues of its 128 R columns in shared memory (PART_BYTES);
// measured slower than W = 1 (profiles/round2_tile512.md), selected only by OZ2_TUNE_TILE_N.
template <int CG, int W = 1>
struct GemmCfg {
    static constexpr int TILE_M = BM * CG;            // output rows per (cluster) tile
    static constexpr int TILE_N = BN * W;             // output columns per tile
    static constexpr int B_ROWS = TILE_N / CG;        // B^T rows staged per CTA
    static constexpr int A_STAGE = BM * BK;
    static constexpr int B_STAGE = B_ROWS * BK;
    static constexpr int NSTAGE = W == 2 ? 3 : CG == 1 ? STAGES : STAGES2;
    static constexpr int PART_BYTES = W == 2 ? 64 * 256 * 4 : 0;   // 64 half2 per epilogue thread
    static constexpr int SMEM = NSTAGE * (A_STAGE + B_STAGE) + 1024 + 256 + static_cast<int>(sizeof(CrtShared)) +
                                16 + PART_BYTES;
};

template <int G>
__device__ __forceinline__ void tile_coords(int t, int m_tiles, int n_tiles, int& tm, int& tn) {
    // groups of G tile-rows swept column by column (oz2_internal.h): G x TILE_M = 2048 rows
    // for both CTA-group sizes
    tile_coords_g(t, G, m_tiles, n_tiles, tm, tn);
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// Relaxed remote arrive: it only contributes an arrival count (the TMA bytes carry their
// own complete_tx, and the TMEM reads it publishes have completed at tcgen05.wait::ld), so
// no release fence is needed -- a .release.cluster arrive costs a MEMBAR per k-stage.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-SM TMA: bytes land in this CTA's smem, completion is counted on the leader's barrier
__device__ __forceinline__ void tma_load_5d_cg2(const CUtensorMap* m, uint32_t leader_bar, void* smem,
                                                int32_t c0, int32_t c1, int32_t c2, int32_t c3, int32_t c4,
                                                uint64_t cache_hint) {
    asm volatile(
        "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;"
        ::"r"(smem_u32(smem)), "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar),
          "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "l"(cache_hint)
        : "memory");
}
// 2-SM TMA multicast: the box lands at the same smem offset in every CTA of `mask`, and
// each destination pair's leader barrier (same offset) counts the bytes
__device__ __forceinline__ void tma_load_5d_cg2_mc(const CUtensorMap* m, uint32_t leader_bar, void* smem,
                                                   int32_t c0, int32_t c1, int32_t c2, int32_t c3, int32_t c4,
                                                   uint16_t mask, uint64_t cache_hint) {
    asm volatile(
        "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
        " [%0], [%1, {%4, %5, %6, %7, %8}], [%2], %3, %9;"
        ::"r"(smem_u32(smem)), "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "h"(mask),
          "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "l"(cache_hint)
        : "memory");
}
__device__ __forceinline__ void mma_f8f6f4_cg2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                               uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void mma_i8_cg2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}
// arrive on the barrier at the same smem offset in every CTA of `mask`
__device__ __forceinline__ void mma_commit_cg2(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
        ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t* dst_smem, uint32_t ncols) {
    if (CG == 1) {
        tmem_alloc(dst_smem, ncols);
    } else {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(dst_smem)), "r"(ncols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t taddr, uint32_t ncols) {
    if (CG == 1) tmem_dealloc(taddr, ncols);
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ constexpr float2 kM2 = {12582912.0f, 12582912.0f};      // 1.5 2^23
__device__ constexpr float2 kNM2 = {-12582912.0f, -12582912.0f};
__device__ constexpr float2 kNM2b = {-8388608.0f, -8388608.0f};     // -2^23

template <int MODE_, int CG, int FL, int MC, int W>
__global__ void __launch_bounds__(GEMM_THREADS, 1)   // 10 warps: 3 on one SM sub-partition -> <= 168 registers
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const __grid_constant__ GemmParams P) {
    // INT8 variants run the same pipeline on kind::i8 (S32 accumulators)
    constexpr bool I8 = MODE_ >= MODE_RESIDUE_I8;
    constexpr int MODE = I8 ? MODE_ - 3 : MODE_;
    // k-block passes per modulus: 3 (FP8: three products, or a K-concatenated pair + one)
    // or 1 (INT8); the number of accumulator drains is P.mod[l].nprod
    constexpr int NP = I8 ? 1 : 3;
    using Cfg = GemmCfg<CG, W>;
    static_assert(W == 1 || (CG == 2 && MC == 1 && MODE_ == MODE_RESIDUE), "256 x 512 tiles: FP8 residue pairs only");
    constexpr int NS = Cfg::NSTAGE;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + NS * Cfg::A_STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + NS * Cfg::B_STAGE);
    uint64_t* empty = full + NS;
    uint64_t* tfull = empty + NS;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    CrtShared* crt_s = reinterpret_cast<CrtShared*>(smem + NS * (Cfg::A_STAGE + Cfg::B_STAGE) + 256);
    // W = 2: partial residues of the R half, [64 pairs][256 epilogue threads] (conflict-free)
    __half2* part_r = reinterpret_cast<__half2*>(
        (reinterpret_cast<uintptr_t>(crt_s) + sizeof(CrtShared) + 15) & ~uintptr_t(15));
    if (FL > 0) crt_stage_constants(crt_s, P.crt, threadIdx.x, blockDim.x);

    const uint32_t warp = warp_id_uniform();
    const uint32_t lane = lane_id();
    // cluster = MC pairs (CG = 2) of CTAs; pairs of one cluster work on horizontally
    // adjacent tiles and share (multicast) the A operand
    constexpr int CS = CG * MC;                                       // cluster size
    const uint32_t crank = (CS > 1) ? cluster_rank() : 0u;
    const uint32_t rank = crank & (CG - 1);                           // rank in the pair
    const uint32_t pairi = crank / CG;                                // pair in the cluster
    const bool leader = rank == 0;
    const uint16_t pair_mask = static_cast<uint16_t>(((1u << CG) - 1u) << (pairi * CG));
    const uint16_t all_mask = static_cast<uint16_t>((1u << CS) - 1u);

    if (warp == 0) {
        if (elect_one()) {
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
            for (int s = 0; s < NS; ++s) {
                mbar_init(&full[s], CG);          // CG = 2: leader expect_tx + peer arrive
                mbar_init(&empty[s], MC);         // one MMA commit per pair reading the stage
            }
            for (int s = 0; s < 2; ++s) {
                mbar_init(&tfull[s], 1);
                mbar_init(&tempty[s], 8 * CG);    // every epilogue warp of the pair
            }
            fence_mbar_init();
        }
        __syncwarp();
    } else if (warp == 1) {
        tmem_alloc_cg<CG>(tmem_slot, 512);
    }
    tc_fence_before();
    // the cluster barrier orders the TMEM-address write of tcgen05.alloc (and the barrier
    // inits) for the whole cluster; the CTA barrier after it changes nothing for the
    // hardware but lets compute-sanitizer racecheck, which does not model barrier.cluster,
    // see the ordering (profiles/round2_sanitizer.md)
    if (CS > 1) cluster_sync_all();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int n_super = P.n_tiles / MC;                  // MC tiles along n per cluster tile
    const int num_tiles = P.m_tiles * n_super;
    const int nkb = P.num_k_blocks;
    // k > 2^16: each product runs as nseg segments of <= 512 k-blocks (2^16 elements), so
    // every FP32 accumulation stays within the exactness window (eq. error-free-FP8-matmult);
    // the epilogue reduces each segment mod p and accumulates the residue (NEXT-2)
    const int nseg = (MODE == MODE_RESIDUE) ? P.num_kseg : 1;
    const int kseg = (MODE == MODE_RESIDUE) ? P.kseg_blocks : nkb;
    // work items: a tile with all its moduli (tile-major, the default), or -- mod_split,
    // for grids with few tiles -- one (tile, modulus) pair, modulus-major over the tiles so
    // that concurrently running units share that modulus' operand panels; the residue of
    // every modulus is independent, only the (then separate) CRT needs them all
    // P.tail_head: tiles [0, head) are tile-major items, tiles [head, num_tiles) are split
    // into (tile, modulus) items (mod_split: head = 0; the hybrid schedule: head = the full
    // waves, so the last partial wave is spread over all units)
    const int head = (MODE == MODE_RESIDUE) ? min(P.tail_head, num_tiles) : num_tiles;
    const int tail = num_tiles - head;
    const int NMOD = (MODE == MODE_RESIDUE) ? P.num_moduli : 1;
    const int num_items = head + tail * NMOD;
    // item -> (tile, first modulus, moduli count)
    auto item_tile = [&](int it) { return it < head ? it : head + (it - head) % tail; };
    auto item_l0 = [&](int it) { return it < head ? 0 : (it - head) / tail; };
    auto item_nmods = [&](int it) { return it < head ? NMOD : 1; };
    // products of modulus l (accumulator drains, each in nseg K segments)
    auto nprod_of = [&](int l) { return (MODE == MODE_RESIDUE) ? P.mod[l].nprod : 1; };
    auto nparts_of = [&](int l, int x) { return (MODE == MODE_RESIDUE && x == 0 && P.mod[l].a_plane2 >= 0) ? 2 : 1; };
    const int unit = blockIdx.x / CS;            // tile-processing unit (cluster)
    const int units = gridDim.x / CS;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (elect_one()) {
            uint32_t stage = 0, phase = 0;
            const uint64_t hint_a = P.hint_a ? P.hint_a : kEvictNormal, hint_b = P.hint_b ? P.hint_b : kEvictNormal;
            long long g = 0;                         // throttle chunks started by this unit
            bool throttle_on = true;
            const long long nunits = units;
            const int kc = P.sync_chunk > 0 ? P.sync_chunk : 1 << 30;   // k-blocks per chunk (power of two)
            const long long chunks_per_prod = (nkb + kc - 1) / kc;
            const uint32_t full0 = smem_u32(&full[0]) & 0xFEFFFFFFu;   // pair leader's barrier (TMA operand)
            const uint32_t full_leader = (CS > 1) ? mapa_shared(smem_u32(&full[0]), crank & ~(CG - 1u)) : 0u;
            for (int it = unit; it < num_items; it += units) {
                const int tile = item_tile(it);
                const int l0 = item_l0(it);
                const int l1 = (MODE == MODE_RESIDUE) ? l0 + item_nmods(it) : l0 + 1;
                int tm, tn;
                tile_coords<16 / CG>(tile, P.m_tiles, n_super, tm, tn);
                tn = tn * MC + static_cast<int>(pairi);
                const int a_row = tm * Cfg::TILE_M + static_cast<int>(rank) * BM + (MC == 2 ? static_cast<int>(pairi) * (BM / 2) : 0);
                const int b_row = tn * Cfg::TILE_N + static_cast<int>(rank) * (BN / CG);
                for (int l = l0; l < l1; ++l)
                for (int x = 0; x < nprod_of(l); ++x)
                for (int seg = 0; seg < nseg; ++seg)
                for (int part = 0; part < nparts_of(l, x); ++part) {
                    // operand planes (interleaved layout: plane = the map's dimension 1)
                    int a_pl = 0, b_pl = 0;
                    int kb0 = 0, kb1 = nkb;
                    if (MODE == MODE_RESIDUE) {
                        a_pl = part ? P.mod[l].a_plane2 : P.mod[l].a_plane[x];
                        b_pl = part ? P.mod[l].b_plane2 : P.mod[l].b_plane[x];
                        kb0 = seg * kseg;
                        kb1 = min(nkb, kb0 + kseg);
                    }
                    for (int kb = kb0; kb < kb1; ++kb) {
                        if (P.sync_lead > 0 && (kb & (kc - 1)) == 0) {     // kc: a power of two
                            // progress throttle: a unit may not run more than sync_lead chunks
                            // (sync_chunk k-blocks each) ahead of the chip-wide average, so
                            // the operand panels streamed by all units stay L2-resident
                            // until every unit sharing them has read them.  It is only a
                            // performance heuristic: a bounded wait (~1 ms) turns it off for
                            // this CTA if other units cannot make progress (e.g. not all
                            // resident), so it can never deadlock.
                            if (crank == 0) atomicAdd(P.progress, 1ull);
                            if (throttle_on) {
                                const long long need = nunits * (g + 1 - P.sync_lead);
                                int spins = 0;
                                while (static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(P.progress)) < need) {
                                    __nanosleep(128);
                                    if (++spins > 8000) { throttle_on = false; break; }
                                }
                            }
                            ++g;
                        }
                        mbar_wait(&empty[stage], phase ^ 1);
                        // map coordinates {K byte in the super-chunk, row in the 128-row block,
                        // plane, super-chunk, row block} (digit planes); a
                        // plain [rows][k] matrix for the raw GEMM: {K byte, row, 0, 0, 0}
                        const int c0 = (kb & ((1 << P.super_shift) - 1)) * BK, c3 = kb >> P.super_shift;
                        const int ar1 = P.row_blocked ? (a_row & (kRowBlk - 1)) : a_row;
                        const int ar4 = P.row_blocked ? (a_row >> 7) : 0;
                        const int br1 = P.row_blocked ? (b_row & (kRowBlk - 1)) : b_row;
                        const int br4 = P.row_blocked ? (b_row >> 7) : 0;
                        if (CG == 1) {
                            mbar_arrive_expect_tx(&full[stage], Cfg::A_STAGE + Cfg::B_STAGE);
                            tma_load_5d(&tmA, &full[stage], sA + stage * Cfg::A_STAGE, c0, ar1, a_pl, c3, ar4, hint_a);
                            tma_load_5d(&tmB, &full[stage], sB + stage * Cfg::B_STAGE, c0, br1, b_pl, c3, br4, hint_b);
                        } else {
                            const uint32_t lb = full0 + stage * 8u;
                            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (Cfg::A_STAGE + Cfg::B_STAGE));
                            else mbar_arrive_cluster(full_leader + stage * 8u);
                            if (MC == 1) {
                                tma_load_5d_cg2(&tmA, lb, sA + stage * Cfg::A_STAGE, c0, ar1, a_pl, c3, ar4, hint_a);
                            } else {
                                // this CTA's half of the A tile, multicast to the CTA with the same
                                // rank in the other pair (which loads the other half for both)
                                const uint16_t amask = static_cast<uint16_t>((1u << rank) | (1u << (rank + CG)));
                                tma_load_5d_cg2_mc(&tmA, lb, sA + stage * Cfg::A_STAGE + pairi * (Cfg::A_STAGE / 2),
                                                   c0, ar1, a_pl, c3, ar4, amask, hint_a);
                            }
                            tma_load_5d_cg2(&tmB, lb, sB + stage * Cfg::B_STAGE, c0, br1, b_pl, c3, br4, hint_b);
                            if (W == 2) {   // this CTA's rows of the R half's B operand (row-blocked maps)
                                const int b2 = b_row + BN;
                                tma_load_5d_cg2(&tmB, lb, sB + stage * Cfg::B_STAGE + (BN / CG) * BK, c0,
                                                b2 & (kRowBlk - 1), b_pl, c3, b2 >> 7, hint_b);
                            }
                        }
                        if (++stage == NS) { stage = 0; phase ^= 1; }
                    }
                }
            }
            if (P.sync_lead > 0 && crank == 0) {
                // finished: count as having started every product so nobody waits on us
                // upper bound of any unit's chunk count (round-robin: <= ceil(head / units)
                // whole-tile items and <= ceil(tail items / units) single-modulus items)
                const long long gmax = (static_cast<long long>((head + units - 1) / units) * (MODE == MODE_RESIDUE ? NP * NMOD * nseg : 1)
                                        + static_cast<long long>((tail * NMOD + units - 1) / units) * NP * nseg)
                                       * chunks_per_prod;
                if (gmax > g) atomicAdd(P.progress, static_cast<unsigned long long>(gmax - g));
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (W == 2 && leader && elect_one()) {
            // 256 x 512 tiles: per K step one N = 256 MMA into each half (L: columns 0-255 of
            // TMEM, R: 256-511), both reading the same staged A.  A product starts its L half as
            // soon as the epilogue has drained L (tempty[0]) and runs it up to NS K steps ahead
            // while R drains; R then catches up and both proceed in lockstep, so the tensor pipe
            // idles only for the part of a drain longer than NS K steps of L MMAs.  tfull[0] is
            // committed after the last L MMA, so L's drain overlaps R's last K steps.
            constexpr uint32_t idesc = make_idesc_e4m3_f32(Cfg::TILE_M, BN);
            uint32_t cnt = 0, g = 0;                 // K steps consumed (ring position), products
            for (int it = unit; it < num_items; it += units) {
                const int l0 = item_l0(it);
                const int l1 = l0 + item_nmods(it);
                for (int l = l0; l < l1; ++l)
                for (int x = 0; x < nprod_of(l); ++x)
                for (int seg = 0; seg < nseg; ++seg, ++g) {
                    const int kb0 = seg * kseg, nk = min(nkb, kb0 + kseg) - kb0;
                    const int nsteps = nparts_of(l, x) * nk;    // (part, k-block) steps
                    auto issue = [&](int s, uint32_t half_col, uint32_t b_off) {
                        const uint32_t q = cnt + static_cast<uint32_t>(s), st = q % NS;
                        const uint64_t a0 = make_desc_k128_sw128(smem_u32(sA + st * Cfg::A_STAGE));
                        const uint64_t b0 = make_desc_k128_sw128(smem_u32(sB + st * Cfg::B_STAGE + b_off));
#pragma unroll
                        for (int kk = 0; kk < BK / 32; ++kk)
                            mma_f8f6f4_cg2(tmem_base + half_col, a0 + 2 * kk, b0 + 2 * kk, idesc,
                                           (s > 0 || kk > 0) ? 1u : 0u);
                    };
                    auto wait_full = [&](int s) {
                        const uint32_t q = cnt + static_cast<uint32_t>(s);
                        mbar_wait(&full[q % NS], (q / NS) & 1u);
                        tc_fence_after();
                    };
                    mbar_wait(&tempty[0], (g & 1u) ^ 1u);
                    tc_fence_after();
                    int sl = 0;
                    for (const int ahead = min(NS, nsteps); sl < ahead; ++sl) {
                        wait_full(sl);
                        issue(sl, 0u, 0u);
                    }
                    if (sl == nsteps) mma_commit_cg2(&tfull[0], pair_mask);
                    mbar_wait(&tempty[1], (g & 1u) ^ 1u);
                    tc_fence_after();
                    for (int sr = 0; sr < nsteps; ++sr) {
                        issue(sr, static_cast<uint32_t>(BN), static_cast<uint32_t>((BN / CG) * BK));
                        mma_commit_cg2(&empty[(cnt + static_cast<uint32_t>(sr)) % NS], pair_mask);
                        if (sl == sr + 1 && sl < nsteps) {          // caught up: lockstep
                            wait_full(sl);
                            issue(sl, 0u, 0u);
                            if (++sl == nsteps) mma_commit_cg2(&tfull[0], pair_mask);
                        }
                    }
                    mma_commit_cg2(&tfull[1], pair_mask);
                    cnt += static_cast<uint32_t>(nsteps);
                }
            }
        } else if (W == 1 && leader && elect_one()) {
            constexpr uint32_t idesc = I8 ? make_idesc_i8_s32(Cfg::TILE_M, BN, MODE != MODE_BOUND)
                                          : make_idesc_e4m3_f32(Cfg::TILE_M, BN);
            uint32_t stage = 0, phase = 0, g = 0;
            for (int it = unit; it < num_items; it += units) {
                const int l0 = item_l0(it);
                const int l1 = (MODE == MODE_RESIDUE) ? l0 + item_nmods(it) : l0 + 1;
                for (int l = l0; l < l1; ++l)
                for (int x = 0; x < nprod_of(l); ++x)
                for (int seg = 0; seg < nseg; ++seg, ++g) {
                    const uint32_t slot = g & 1u, use = g >> 1;
                    mbar_wait(&tempty[slot], (use & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + slot * BN;
                    const int kb0 = seg * kseg, kb1 = min(nkb, kb0 + kseg);
                    const int nparts = nparts_of(l, x);
                    for (int part = 0; part < nparts; ++part)
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint64_t a0 = make_desc_k128_sw128(smem_u32(sA + stage * Cfg::A_STAGE));
                        const uint64_t b0 = make_desc_k128_sw128(smem_u32(sB + stage * Cfg::B_STAGE));
#pragma unroll
                        for (int kk = 0; kk < BK / 32; ++kk) {
                            // advance 32 bytes of K inside the 128-byte swizzle atom
                            const uint32_t acc = (part > 0 || kb > kb0 || kk > 0) ? 1u : 0u;
                            if (I8) {
                                if (CG == 1) mma_i8(d_tmem, a0 + 2 * kk, b0 + 2 * kk, idesc, acc);
                                else mma_i8_cg2(d_tmem, a0 + 2 * kk, b0 + 2 * kk, idesc, acc);
                            } else {
                                if (CG == 1) mma_f8f6f4(d_tmem, a0 + 2 * kk, b0 + 2 * kk, idesc, acc);
                                else mma_f8f6f4_cg2(d_tmem, a0 + 2 * kk, b0 + 2 * kk, idesc, acc);
                            }
                        }
                        if (CG == 1) mma_commit(&empty[stage]);
                        else mma_commit_cg2(&empty[stage], MC == 2 ? all_mask : pair_mask);
                        if (++stage == NS) { stage = 0; phase ^= 1; }
                    }
                    if (CG == 1) mma_commit(&tfull[slot]);
                    else mma_commit_cg2(&tfull[slot], pair_mask);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const uint32_t quad = warp & 3u;           // TMEM lane quadrant this warp may access
        const uint32_t half = (warp - 2u) >> 2;    // 128-column half of the 256-column tile
        const uint32_t row_in_tile = rank * BM + quad * 32u + lane;
        const uint32_t tempty0 = (CG == 2) ? mapa_shared(smem_u32(&tempty[0]), crank & ~(CG - 1u)) : 0u;
        auto release_slot = [&](uint32_t slot) {
            // accumulator slot drained: hand it back to the (leader's) MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 1) mbar_arrive(&tempty[slot]);
                else mbar_arrive_cluster(tempty0 + slot * 8u);
            }
        };
        // Fused CRT + inverse scaling (FL > 0): a finished tile's CRT is spread over the
        // products of the next tile, crt_per_prod columns after each product, so its
        // residue loads never delay the release of an accumulator slot.  The N residues
        // of an element were written by this same thread (program order).
        // A thread's columns of a tile: 128 (W = 1), or 128 of the L half and the same 128 of
        // the R half, BN columns further (W = 2).
        constexpr int TCOLS = 128 * W;
        int64_t crt_row = -1, crt_col0 = 0;
        int crt_j = TCOLS;
        const int crt_per_prod = (MODE == MODE_RESIDUE) ? (TCOLS + P.prods_per_tile * nseg - 1) / (P.prods_per_tile * nseg) + 1 : 0;
        auto crt_steps = [&](int ncols) {
            if (FL == 0 || crt_j >= TCOLS) return;
            if (crt_row >= P.m) { crt_j = TCOLS; return; }
            const int emu = P.e_mu[crt_row];
            const int64_t lstride = static_cast<int64_t>(P.n) * P.m;
#pragma unroll 1
            for (int s2 = 0; s2 < ncols && crt_j < TCOLS; ++s2, ++crt_j) {
                const int64_t col = crt_col0 + crt_j + (W == 2 && crt_j >= 128 ? BN - 128 : 0);
                if (col >= P.n) { crt_j = TCOLS; break; }   // (R columns lie right of L's)
                const int enu = P.e_nu[col];
                const double v = exps_finite(emu, enu)
                                     ? crt_element<(FL > 0 ? FL : 4)>(P.residues + col * P.m + crt_row, lstride,
                                                                      crt_s, P.crt, emu + enu, true)
                                     : __longlong_as_double(0x7FF8000000000000ll);      // R12
                store_alpha_beta(P.C + crt_row + col * P.ldc, v, P.alpha, P.beta);
            }
        };
        uint32_t g = 0;
        const uint32_t et = threadIdx.x - 64u;    // epilogue thread index (W = 2 partials)
        for (int it = unit; it < num_items; it += units) {
            const int tile = item_tile(it);
            const int l0 = item_l0(it);
            const int mods_per_item = item_nmods(it);
            int tm, tn;
            tile_coords<16 / CG>(tile, P.m_tiles, n_super, tm, tn);
            tn = tn * MC + static_cast<int>(pairi);
            const int64_t row = static_cast<int64_t>(tm) * Cfg::TILE_M + row_in_tile;
            const int64_t col0 = static_cast<int64_t>(tn) * Cfg::TILE_N + half * 128u;
            const bool row_ok = row < P.m;
            if (W == 2) {
                // 256 x 512 tile: per product drain L (columns col0 + [0, 128)), release it,
                // then R (col0 + BN + [0, 128)); partial residues of L in registers, of R in
                // shared memory.  Same arithmetic as the W = 1 epilogue below.
                for (int l = l0; l < l0 + mods_per_item; ++l) {
                    const float p = P.mod[l].p, pinv = P.mod[l].pinv;
                    __half2 part[64];
                    int16_t* outL = P.residues + (static_cast<int64_t>(l) * P.n + col0) * P.m + row;
                    const int npl = nprod_of(l);
                    for (int x = 0; x < npl; ++x) {
                      const float coef = P.mod[l].coef[x];
                      for (int seg = 0; seg < nseg; ++seg, ++g) {
                        const bool first = (x == 0) && (seg == 0);
                        const bool last = (x == npl - 1) && (seg == nseg - 1);
                        auto drain = [&](auto RIGHT) {
                            constexpr bool R = decltype(RIGHT)::value;
                            const uint32_t slot = R ? 1u : 0u;
                            if (P.epi_sleep_ns) mbar_wait_sleep(&tfull[slot], g & 1u, P.epi_sleep_ns);
                            else mbar_wait(&tfull[slot], g & 1u);
                            tc_fence_after();
                            const int64_t cb = col0 + (R ? BN : 0);
                            int16_t* out = outL + (R ? static_cast<int64_t>(BN) * P.m : 0);
                            const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + slot * BN + half * 128u;
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                uint32_t v[32];
                                tmem_ld_32x32b_x32(taddr + c * 32, v);
                                tmem_ld_wait();
                                if (c == 3) release_slot(slot);
                                const bool chunk_full = row_ok && cb + c * 32 + 32 <= P.n;
#pragma unroll
                                for (int j = 0; j < 32; j += 2) {
                                    const float2 f = make_float2(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
                                    const float2 pinv2 = make_float2(pinv, pinv), np2 = make_float2(-p, -p);
                                    float2 q = __fadd2_rn(__ffma2_rn(f, pinv2, kM2), kNM2);
                                    float2 a2 = __ffma2_rn(q, np2, f);
                                    const int idx = (c * 32 + j) >> 1;
                                    const float2 cf = make_float2(coef, coef);
                                    if (first) a2 = __fmul2_rn(a2, cf);
                                    else a2 = __ffma2_rn(a2, cf, __half22float2(R ? part_r[idx * 256 + et] : part[idx]));
                                    q = __fadd2_rn(__ffma2_rn(a2, pinv2, kM2), kNM2);
                                    a2 = __ffma2_rn(q, np2, a2);
                                    if (!last) {
                                        const __half2 h = __floats2half2_rn(a2.x, a2.y);   // exact (|.| <= 546)
                                        if (R) part_r[idx * 256 + et] = h;
                                        else part[idx] = h;
                                    } else {
                                        const float2 u2 = __fadd2_rn(make_float2(a2.x < 0.0f ? a2.x + p : a2.x,
                                                                                 a2.y < 0.0f ? a2.y + p : a2.y),
                                                                     make_float2(8388608.0f, 8388608.0f));
                                        const int jj = c * 32 + j;
                                        int16_t* o = out + static_cast<int64_t>(jj) * P.m;
                                        if (chunk_full) {
                                            __stcs(o, static_cast<short>(__float_as_int(u2.x)));
                                            __stcs(o + P.m, static_cast<short>(__float_as_int(u2.y)));
                                        } else if (row_ok) {
                                            if (cb + jj < P.n) __stcs(o, static_cast<short>(__float_as_int(u2.x)));
                                            if (cb + jj + 1 < P.n) __stcs(o + P.m, static_cast<short>(__float_as_int(u2.y)));
                                        }
                                    }
                                }
                            }
                        };
                        drain(std::integral_constant<bool, false>());
                        drain(std::integral_constant<bool, true>());
                        crt_steps(crt_per_prod);
                      }
                    }
                }
                if (FL > 0 && it < head) {   // split tail items: their CRT runs in k_crt_tiles
                    crt_steps(TCOLS);
                    crt_row = row;
                    crt_col0 = col0;
                    crt_j = 0;
                }
            } else if (MODE == MODE_RESIDUE) {
                for (int l = l0; l < l0 + mods_per_item; ++l) {
                    const float p = P.mod[l].p, pinv = P.mod[l].pinv, w16 = P.mod[l].w16;
                    // running partial sum_x coef_x r_x, reduced mod p after every product
                    // (|.| <= p/2 + 1 <= 546), held exactly in binary16 pairs
                    __half2 part[64];
                    int16_t* out = P.residues + (static_cast<int64_t>(l) * P.n + col0) * P.m + row;
                    const int npl = nprod_of(l);
                    for (int x = 0; x < npl; ++x) {
                      const float coef = P.mod[l].coef[x];
                      for (int seg = 0; seg < nseg; ++seg, ++g) {
                        const bool first = (x == 0) && (seg == 0);
                        const bool last = (x == npl - 1) && (seg == nseg - 1);
                        const uint32_t slot = g & 1u, use = g >> 1;
                        // the other slot's product is still running: no hurry (the MMAs of
                        // product g+2 need this slot only after product g+1, ~60 us away)
                        if (P.epi_sleep_ns) mbar_wait_sleep(&tfull[slot], use & 1u, P.epi_sleep_ns);
                        else mbar_wait(&tfull[slot], use & 1u);
                        tc_fence_after();
                        const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + slot * BN + half * 128u;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            uint32_t v[32];
                            tmem_ld_32x32b_x32(taddr + c * 32, v);
                            tmem_ld_wait();
                            if (c == 3) release_slot(slot);   // the whole slot is in registers
                            const bool chunk_full = row_ok && col0 + c * 32 + 32 <= P.n;
#pragma unroll
                            for (int j = 0; j < 32; j += 2) {
                                // packed FP32 pairs; x - p rint(x/p) by the 1.5 2^23 magic-number
                                // rounding of one FFMA2 (exact: |x/p| < 2^22)
                                float2 f;
                                if (I8) {
                                    // S32 sum (|.| <= 2^30) == hi w16 + lo (mod p): both halves
                                    // exact floats via the 2^23 exponent trick, |f| < 2^23
                                    const int i0 = static_cast<int>(v[j]), i1 = static_cast<int>(v[j + 1]);
                                    const float2 hi = __fadd2_rn(make_float2(__int_as_float(0x4B400000 + (i0 >> 16)),
                                                                             __int_as_float(0x4B400000 + (i1 >> 16))), kNM2);
                                    const float2 lo = __fadd2_rn(make_float2(__int_as_float(0x4B000000 | (i0 & 0xFFFF)),
                                                                             __int_as_float(0x4B000000 | (i1 & 0xFFFF))), kNM2b);
                                    f = __ffma2_rn(hi, make_float2(w16, w16), lo);
                                } else {
                                    f = make_float2(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));   // exact, <= 2^24
                                }
                                const float2 pinv2 = make_float2(pinv, pinv), np2 = make_float2(-p, -p);
                                float2 q = __fadd2_rn(__ffma2_rn(f, pinv2, kM2), kNM2);
                                float2 a2 = __ffma2_rn(q, np2, f);
                                const int idx = (c * 32 + j) >> 1;
                                const float2 cf = make_float2(coef, coef);
                                if (first) a2 = __fmul2_rn(a2, cf);
                                else a2 = __ffma2_rn(a2, cf, __half22float2(part[idx]));
                                q = __fadd2_rn(__ffma2_rn(a2, pinv2, kM2), kNM2);
                                a2 = __ffma2_rn(q, np2, a2);
                                float acc[2] = {a2.x, a2.y};
                                if (!last) {
                                    part[idx] = __floats2half2_rn(acc[0], acc[1]);  // exact (|acc| <= 546)
                                } else {
                                    // C'_l mod p stored as u in [0, p) (|acc| <= p/2 + 1 here);
                                    // the CRT consumes u directly, the debug output converts
                                    // it back to the symmetric range (R2).  u + 2^23 holds u in
                                    // its low bits (no float-to-int conversion).
                                    const float2 u2 = __fadd2_rn(make_float2(acc[0] < 0.0f ? acc[0] + p : acc[0],
                                                                             acc[1] < 0.0f ? acc[1] + p : acc[1]),
                                                                 make_float2(8388608.0f, 8388608.0f));
                                    const int jj = c * 32 + j;
                                    int16_t* o = out + static_cast<int64_t>(jj) * P.m;   // streamed: read once by the CRT
                                    if (chunk_full) {
                                        __stcs(o, static_cast<short>(__float_as_int(u2.x)));
                                        __stcs(o + P.m, static_cast<short>(__float_as_int(u2.y)));
                                    } else if (row_ok) {
                                        if (col0 + jj < P.n) __stcs(o, static_cast<short>(__float_as_int(u2.x)));
                                        if (col0 + jj + 1 < P.n) __stcs(o + P.m, static_cast<short>(__float_as_int(u2.y)));
                                    }
                                }
                            }
                        }
                        crt_steps(crt_per_prod);
                      }
                    }
                }
                if (FL > 0 && it < head) {   // split tail items: their CRT runs in k_crt_tiles
                    crt_steps(TCOLS);             // finish the previous tile if still pending
                    crt_row = row;                // this tile's CRT is spread over the next tile
                    crt_col0 = col0;
                    crt_j = 0;
                }
            } else {
                const uint32_t slot = g & 1u, use = g >> 1;
                if (P.epi_sleep_ns) mbar_wait_sleep(&tfull[slot], use & 1u, P.epi_sleep_ns);
                else mbar_wait(&tfull[slot], use & 1u);
                tc_fence_after();
                const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + slot * BN + half * 128u;
                // non-negative FP32 and S32 values both order like their bit patterns
                uint32_t rowmax = 0u;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(taddr + c * 32, v);
                    tmem_ld_wait();
                    if (MODE == MODE_BOUND) {
                        uint32_t mycol = 0;
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            rowmax = max(rowmax, v[j]);
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
                release_slot(slot);
                ++g;
                if (MODE == MODE_BOUND && row < P.m && rowmax > 0u)
                    atomicMax(P.rmax + row, rowmax);
            }
        }
        crt_steps(TCOLS);                         // the last tile's CRT
    }

    tc_fence_before();
    if (CS > 1) cluster_sync_all();
    else __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc_cg<CG>(tmem_base, 512);
    }
}

constexpr int kMaxDevices = 64;

template <int MODE, int CG, int FL, int MC, int W = 1>
static cudaError_t launch_one(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& gp,
                              int num_sms, cudaStream_t st) {
    using Cfg = GemmCfg<CG, W>;
    constexpr int CS = CG * MC;
    const int num_tiles = gp.m_tiles * (gp.n_tiles / MC);
    if (num_tiles == 0) return cudaSuccess;
    const bool res_mode = MODE == MODE_RESIDUE || MODE == MODE_RESIDUE_I8;
    const int head = res_mode ? (gp.tail_head < num_tiles ? gp.tail_head : num_tiles) : num_tiles;
    const int num_items = head + (num_tiles - head) * (res_mode ? gp.num_moduli : 1);
    // kernel attributes and the co-resident cluster count, once per device (attributes are
    // per device; several host threads may launch concurrently)
    static std::mutex mu;
    static int max_clusters_dev[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu);
    int& max_clusters = max_clusters_dev[dev];
    if (max_clusters == 0) {
        cudaError_t err = cudaFuncSetAttribute(gemm_kernel<MODE, CG, FL, MC, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        if (err != cudaSuccess) return err;
        if (CS > 1) {
            err = cudaFuncSetAttribute(gemm_kernel<MODE, CG, FL, MC, W>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3((num_sms / CS) * CS);
            q.blockDim = dim3(GEMM_THREADS);
            q.dynamicSmemBytes = Cfg::SMEM;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = CS;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, gemm_kernel<MODE, CG, FL, MC, W>, &q) != cudaSuccess || nc <= 0) {
                cudaGetLastError();
                nc = num_sms / CS;
            }
            max_clusters = nc;
        } else {
            max_clusters = num_sms;
        }
    }
    // persistent grid: never more units than can be resident at once (the progress
    // throttle assumes every unit runs concurrently)
    int max_units = num_sms / CS;
    if (max_clusters < max_units) max_units = max_clusters;
    // OZ2_TUNE_MAX_UNITS: experiment knob, caps the persistent units (power-wall study)
    if (gp.max_units > 0 && gp.max_units < max_units) max_units = gp.max_units;
    const int units = num_items < max_units ? num_items : max_units;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(units * CS);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, gemm_kernel<MODE, CG, FL, MC, W>, ta, tb, gp);
}

template <int CG, int MC>
static cudaError_t launch_cg(int mode, int fl, const CUtensorMap& ta, const CUtensorMap& tb,
                            const GemmParams& gp, int num_sms, cudaStream_t st) {
    if (mode == MODE_BOUND) return launch_one<MODE_BOUND, CG, 0, MC>(ta, tb, gp, num_sms, st);
    if (mode == MODE_RAW) return launch_one<MODE_RAW, CG, 0, MC>(ta, tb, gp, num_sms, st);
    if (MC == 1) {   // INT8 scheme: CTA-pair (CG = 2) and single-CTA tiles
        if (mode == MODE_BOUND_I8) return launch_one<MODE_BOUND_I8, CG, 0, MC>(ta, tb, gp, num_sms, st);
        if (mode == MODE_RAW_I8) return launch_one<MODE_RAW_I8, CG, 0, MC>(ta, tb, gp, num_sms, st);
        if (mode == MODE_RESIDUE_I8) {
            switch (fl) {
                case 4: return launch_one<MODE_RESIDUE_I8, CG, 4, MC>(ta, tb, gp, num_sms, st);
                case 5: return launch_one<MODE_RESIDUE_I8, CG, 5, MC>(ta, tb, gp, num_sms, st);
                case 6: return launch_one<MODE_RESIDUE_I8, CG, 6, MC>(ta, tb, gp, num_sms, st);
                default: return launch_one<MODE_RESIDUE_I8, CG, 0, MC>(ta, tb, gp, num_sms, st);
            }
        }
    } else if (mode >= MODE_RESIDUE_I8) {
        return cudaErrorInvalidValue;
    }
    switch (fl) {
        case 4: return launch_one<MODE_RESIDUE, CG, 4, MC>(ta, tb, gp, num_sms, st);
        case 5: return launch_one<MODE_RESIDUE, CG, 5, MC>(ta, tb, gp, num_sms, st);
        case 6: return launch_one<MODE_RESIDUE, CG, 6, MC>(ta, tb, gp, num_sms, st);
        default: return launch_one<MODE_RESIDUE, CG, 0, MC>(ta, tb, gp, num_sms, st);
    }
}

// cg = 1: 128x256 single-CTA tiles; cg = 2: 256x256 CTA pairs; cg = 4: clusters of two
// pairs on horizontally adjacent tiles sharing A by TMA multicast (needs even n_tiles);
// tile_n = 512 (cg = 2, FP8 residue mode): 256x512 CTA-pair tiles (gp.n_tiles in 512-column units)
cudaError_t launch_gemm(int mode, int cg, int fused_limbs, const CUtensorMap& ta, const CUtensorMap& tb,
                        const GemmParams& gp, int num_sms, cudaStream_t st, int tile_n) {
    cudaError_t err;
    if (tile_n == 512) {
        if (cg != 2 || mode != MODE_RESIDUE) return cudaErrorInvalidValue;
        switch (fused_limbs) {
            case 4: err = launch_one<MODE_RESIDUE, 2, 4, 1, 2>(ta, tb, gp, num_sms, st); break;
            case 5: err = launch_one<MODE_RESIDUE, 2, 5, 1, 2>(ta, tb, gp, num_sms, st); break;
            case 6: err = launch_one<MODE_RESIDUE, 2, 6, 1, 2>(ta, tb, gp, num_sms, st); break;
            default: err = launch_one<MODE_RESIDUE, 2, 0, 1, 2>(ta, tb, gp, num_sms, st); break;
        }
    } else if (cg == 4 && mode < MODE_RESIDUE_I8) err = launch_cg<2, 2>(mode, fused_limbs, ta, tb, gp, num_sms, st);
    else if (cg == 4) return cudaErrorInvalidValue;       // no multicast variant of the kind::i8 kernels
    else if (cg == 2) err = launch_cg<2, 1>(mode, fused_limbs, ta, tb, gp, num_sms, st);
    else err = launch_cg<1, 1>(mode, fused_limbs, ta, tb, gp, num_sms, st);
    if (err != cudaSuccess) return err;
    return cudaGetLastError();
}

}  // namespace oz2
