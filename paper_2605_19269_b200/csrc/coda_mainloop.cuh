// coda_mainloop.cuh — the fixed GEMM mainloop shared by every CODA kernel.
//
// Persistent tile loop over output tiles (raster groups of m-tiles for L2
// reuse), a multi-stage TMA -> smem ring of 64-wide k-blocks in SWIZZLE_128B
// layout, and a single-thread tcgen05.mma issuer accumulating in TMEM with two
// accumulator buffers so the epilogue of tile i overlaps the mainloop of i+1.
//
// CG = 1: one CTA computes a 128 x 256 tile (tcgen05.mma.cta_group::1, M=128).
// CG = 2: a cluster of two CTAs computes a 256 x 256 tile with
//   tcgen05.mma.cta_group::2 (M=256) issued by the leader (rank 0).  Each CTA
//   loads its own 128 rows of A and one 128-column half of B; the 2-SM TMA
//   loads count their bytes on the leader's barrier; commits are multicast to
//   both CTAs; each CTA's TMEM holds its 128 rows x 256 columns.  Halves the
//   per-SM shared-memory and L2 traffic of the B operand.
#pragma once
#include <cstdint>
#include <cuda.h>
#include "coda_ptx.cuh"

namespace coda {

constexpr int BM = 128;                      // accumulator rows per CTA (TMEM lanes)
constexpr int BN = 256;                      // accumulator columns per tile
constexpr int BK = 64;                       // one 128-byte swizzle atom of bf16 along K
constexpr int STAGES = 4;                    // CG = 1 ring depth (48 KiB stages)
constexpr int A_STAGE_BYTES = BM * BK * 2;   // 16 KiB
constexpr int B_STAGE_BYTES = BN * BK * 2;   // 32 KiB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int TMEM_COLS = 512;               // 2 accumulator buffers x 256 columns

template <int CG>
struct Geom {
    static constexpr int TILE_M = BM * CG;                 // rows per (pair) tile
    static constexpr int B_COLS = BN / CG;                 // B columns loaded per CTA
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = B_COLS * BK * 2;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int NSTAGE = CG == 1 ? 4 : 6;         // 192 KiB of operand ring either way
    static constexpr int RING = NSTAGE * STAGE;
};

struct MainParams {
    int M, N, K;
    int ntm, ntn, nk, ntiles;   // ntm counts (pair) tiles of Geom<CG>::TILE_M rows
    int a_mn, b_mn;             // operand majorness: 1 = MN-major (transposed storage)
    int group;                  // raster group: m-tiles swept together across all n-tiles
    // Tail splitting (wave quantization): the last `tail` tiles are split along K into
    // `split` pieces that run concurrently in the final round; work items are the
    // `full_tiles` whole tiles followed by tail x split pieces.
    int full_tiles, tail, split, nitems;
    int prefetch;               // L2 prefetch distance in k-blocks beyond the load (0 = off)
    int ns;                     // ring stages in use (<= the compiled ring depth; 0 = all)
#ifdef CODA_EXPERIMENTS
    // Soft wave barrier (0 = off): a producer arrives on the wave's counter once its tile
    // has issued `wave_pct` % of its k-blocks, and holds the next wave's first load until
    // every producer of the launch has arrived (bounded wait: a hint, never a dependency),
    // keeping the CTAs that share operand panels within a tile of each other in K.
    int wave_pct;
    int* wave_ctr;              // [waves] counters + a finish counter, zero between launches
#endif
};

// One unit of scheduled work: a whole tile (piece = -1) or piece `piece` of tail tile `tail_idx`.
struct Work {
    int tm, tn, kb0, kb1, piece, tail_idx;
};

__device__ __forceinline__ void tile_coord(const MainParams& mp, int t, int& tm, int& tn);

__device__ __forceinline__ Work work_item(const MainParams& mp, int i) {
    Work w;
    int t;
    if (i < mp.full_tiles) {
        t = i;
        w.piece = -1;
        w.tail_idx = -1;
        w.kb0 = 0;
        w.kb1 = mp.nk;
    } else {
        const int j = i - mp.full_tiles;
        w.tail_idx = j / mp.split;
        w.piece = j - w.tail_idx * mp.split;
        t = mp.full_tiles + w.tail_idx;
        w.kb0 = (int)((int64_t)w.piece * mp.nk / mp.split);
        w.kb1 = (int)((int64_t)(w.piece + 1) * mp.nk / mp.split);
    }
    tile_coord(mp, t, w.tm, w.tn);
    return w;
}

__device__ __forceinline__ void tile_coord(const MainParams& mp, int t, int& tm, int& tn) {
    const int per_group = mp.group * mp.ntn;
    const int g = t / per_group;
    const int first = g * mp.group;
    const int gs = min(mp.ntm - first, mp.group);
    const int r = t - g * per_group;
    tm = first + r % gs;
    tn = r / gs;
}

// TMA producer (one warp per CTA, warp-uniform control flow; one elected lane
// issues): fills this CTA's smem ring for every tile it owns.
template <int CG, int NS = Geom<CG>::NSTAGE>
__device__ __forceinline__ void producer_loop(const MainParams& mp, const CUtensorMap* tma_a,
                                              const CUtensorMap* tma_b, uint8_t* sA, uint8_t* sB,
                                              uint64_t* full, uint64_t* empty, int rank, int unit, int nunits) {
    using G = Geom<CG>;
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t sa0 = smem_u32(sA), sb0 = smem_u32(sB);
    const int nst = (mp.ns > 0 && mp.ns < NS) ? mp.ns : NS;
    auto boxes = [&](auto&& op, int m0, int nb0, int kb) {
        const int k0 = kb * BK;
        if (!mp.a_mn) {
            op(0, tma_a, k0, m0);
        } else {
#pragma unroll
            for (int b = 0; b < BM / 64; ++b) op(b * (BK * 128), tma_a, m0 + 64 * b, k0);
        }
        if (!mp.b_mn) {
            op(-1, tma_b, k0, nb0);
        } else {
#pragma unroll
            for (int b = 0; b < G::B_COLS / 64; ++b) op(-1 - b * (BK * 128), tma_b, nb0 + 64 * b, k0);
        }
    };
    auto prefetch = [&](int, const CUtensorMap* map, int c0, int c1) { tma_prefetch_2d(map, c0, c1); };
    const int pf = mp.prefetch;
    if (pf > 0 && unit < mp.nitems && elect_one()) {
        // warm L2 for the first k-blocks this unit will load beyond the ring
        const Work w = work_item(mp, unit);
        const int m0 = w.tm * G::TILE_M + rank * BM, nb0 = w.tn * BN + rank * G::B_COLS;
        for (int kb = w.kb0 + nst; kb < w.kb1 && kb < w.kb0 + nst + pf; ++kb) boxes(prefetch, m0, nb0, kb);
    }
    __syncwarp();
#ifdef CODA_EXPERIMENTS
    const bool wsync = mp.wave_pct > 0 && mp.wave_ctr != nullptr;
    const int producers = nunits * CG;
#endif
    for (int i = unit; i < mp.nitems; i += nunits) {
        const Work w = work_item(mp, i);
        const int m0 = w.tm * G::TILE_M + rank * BM;
        const int nb0 = w.tn * BN + rank * G::B_COLS;
#ifdef CODA_EXPERIMENTS
        const int wave = (i - unit) / nunits;
        if (wsync && wave > 0 && w.piece < 0) {
            // bounded wait for every producer to pass the previous wave's milestone
            if (elect_one()) {
                const int* c = mp.wave_ctr + (wave - 1);
                for (int it = 0; it < 400; ++it) {
                    int v;
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
                    if (v >= producers) break;
                    __nanosleep(64);
                }
            }
            __syncwarp();
        }
        const int milestone = w.kb0 + (int)((int64_t)(w.kb1 - w.kb0) * mp.wave_pct / 100);
#endif
        // the item after this one (prefetch target once this item's k-blocks run out)
        const bool has_next = i + nunits < mp.nitems;
        Work wn = w;
        if (pf > 0 && has_next) wn = work_item(mp, i + nunits);
        const int m0n = wn.tm * G::TILE_M + rank * BM, nb0n = wn.tn * BN + rank * G::B_COLS;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
#ifdef CODA_EXPERIMENTS
            if (wsync && w.piece < 0 && kb == milestone && elect_one())
                atomicAdd(mp.wave_ctr + wave, 1);
#endif
            mbar_wait(&empty[stage], phase ^ 1);
            if (elect_one()) {
                if (rank == 0) mbar_arrive_expect_tx(&full[stage], G::STAGE * CG);
                const uint32_t sa = sa0 + stage * G::A_BYTES;
                const uint32_t sb = sb0 + stage * G::B_BYTES;
                uint64_t* bar = &full[stage];
                auto load = [&](int off, const CUtensorMap* map, int c0, int c1) {
                    const uint32_t dst = off >= 0 ? sa + (uint32_t)off : sb + (uint32_t)(-1 - off);
                    if constexpr (CG == 1) tma_load_2d(dst, map, c0, c1, bar);
                    else tma_load_2d_pair(dst, map, c0, c1, bar);
                };
                boxes(load, m0, nb0, kb);
                if (pf > 0) {
                    // keep L2 `pf` k-blocks ahead of the ring: this item, then the next one
                    const int kp = kb + nst + pf;
                    if (kp < w.kb1) boxes(prefetch, m0, nb0, kp);
                    else if (has_next && kp - w.kb1 + wn.kb0 < wn.kb1) boxes(prefetch, m0n, nb0n, kp - w.kb1 + wn.kb0);
                }
            }
            __syncwarp();
            if (++stage == nst) { stage = 0; phase ^= 1; }
        }
    }
#ifdef CODA_EXPERIMENTS
    if (wsync && elect_one()) {
        // the last producer to finish clears the counters for the next launch
        const int nw = (mp.nitems + nunits - 1) / nunits;
        int* fin = mp.wave_ctr + nw;
        if (atomicAdd(fin, 1) == producers - 1) {
            for (int k = 0; k <= nw; ++k) mp.wave_ctr[k] = 0;
            __threadfence();
        }
    }
    __syncwarp();
#endif
}

// MMA issuer (one warp; for CG = 2 only in the leader CTA; one elected lane issues):
// 4 x tcgen05.mma (K = 16 each) per k-block into the current TMEM accumulator;
// commits free smem stages and publish finished accumulators.  Descriptors are a
// per-launch base plus compile-time/stage offsets in the 14-bit address field
// (smem addresses < 256 KiB, so the field never carries).
template <int CG, int NS = Geom<CG>::NSTAGE>
__device__ __forceinline__ void mma_loop(const MainParams& mp, uint32_t tmem_base, uint8_t* sA, uint8_t* sB,
                                         uint64_t* full, uint64_t* empty, uint64_t* tfull, uint64_t* tempty,
                                         int unit, int nunits) {
    using G = Geom<CG>;
    // kind::f16 instruction descriptor: D f32, A/B bf16, majorness, N>>3, M>>4.
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)mp.a_mn << 15) |
                           ((uint32_t)mp.b_mn << 16) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(G::TILE_M >> 4) << 24);
    // K-major: LBO unused (16), SBO = 8 rows * 128 B; advance 32 B per UMMA_K = 16.
    // MN-major: LBO = next 64-wide MN atom column (BK * 128 B), SBO = 8 K-rows * 128 B;
    //           advance 2 x 1024 B per UMMA_K = 16.
    const uint32_t a_lbo = mp.a_mn ? BK * 128 : 16, b_lbo = mp.b_mn ? BK * 128 : 16;
    const uint64_t a_step = mp.a_mn ? (2048 >> 4) : (32 >> 4), b_step = mp.b_mn ? (2048 >> 4) : (32 >> 4);
    const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA), a_lbo, 1024);
    const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sB), b_lbo, 1024);
    const int nst = (mp.ns > 0 && mp.ns < NS) ? mp.ns : NS;
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int i = unit; i < mp.nitems; i += nunits) {
        const Work w = work_item(mp, i);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (elect_one()) {
                const uint64_t ad = a_desc0 + (uint64_t)((stage * G::A_BYTES) >> 4);
                const uint64_t bd = b_desc0 + (uint64_t)((stage * G::B_BYTES) >> 4);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    const uint32_t accum = (kb != w.kb0 || k != 0) ? 1u : 0u;
                    if constexpr (CG == 1) umma_bf16(d_tmem, ad + k * a_step, bd + k * b_step, idesc, accum);
                    else umma_bf16_pair(d_tmem, ad + k * a_step, bd + k * b_step, idesc, accum);
                }
                if constexpr (CG == 1) umma_commit(&empty[stage]);
                else umma_commit_pair(&empty[stage]);
            }
            __syncwarp();
            if (++stage == nst) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) {
            if constexpr (CG == 1) umma_commit(&tfull[acc]);
            else umma_commit_pair(&tfull[acc]);
        }
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
    }
}

}  // namespace coda
