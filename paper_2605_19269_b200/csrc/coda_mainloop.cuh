// coda_mainloop.cuh — the fixed GEMM mainloop shared by every CODA kernel.
//
// Persistent tile loop over 128 x 256 output tiles (raster groups of 16
// m-tiles for L2 reuse of the B panel), a 4-stage TMA -> smem ring of 64-wide
// k-blocks in SWIZZLE_128B layout, and a single-thread tcgen05.mma issuer
// accumulating in TMEM with two accumulator buffers so the epilogue of tile i
// overlaps the mainloop of tile i+1.
#pragma once
#include <cstdint>
#include <cuda.h>
#include "coda_ptx.cuh"

namespace coda {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;                       // one 128-byte swizzle atom of bf16 along K
constexpr int STAGES = 4;
constexpr int A_STAGE_BYTES = BM * BK * 2;   // 16 KiB
constexpr int B_STAGE_BYTES = BN * BK * 2;   // 32 KiB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int TMEM_COLS = 512;               // 2 accumulator buffers x 256 columns
constexpr int RASTER_GROUP = 16;             // m-tiles per raster group (L2 reuse)

struct MainParams {
    int M, N, K;
    int ntm, ntn, nk, ntiles;
    int a_mn, b_mn;      // operand majorness: 1 = MN-major (transposed storage)
};

__device__ __forceinline__ void tile_coord(const MainParams& mp, int t, int& tm, int& tn) {
    const int per_group = RASTER_GROUP * mp.ntn;
    const int g = t / per_group;
    const int first = g * RASTER_GROUP;
    const int gs = min(mp.ntm - first, RASTER_GROUP);
    const int r = t - g * per_group;
    tm = first + r % gs;
    tn = r / gs;
}

// TMA producer (one thread): fills the smem ring for every tile this CTA owns.
__device__ __forceinline__ void producer_loop(const MainParams& mp, const CUtensorMap* tma_a,
                                              const CUtensorMap* tma_b, uint8_t* sA, uint8_t* sB,
                                              uint64_t* full, uint64_t* empty) {
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < mp.ntiles; t += gridDim.x) {
        int tm, tn;
        tile_coord(mp, t, tm, tn);
        const int m0 = tm * BM, n0 = tn * BN;
        for (int kb = 0; kb < mp.nk; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
            const uint32_t sa = smem_u32(sA + stage * A_STAGE_BYTES);
            const uint32_t sb = smem_u32(sB + stage * B_STAGE_BYTES);
            const int k0 = kb * BK;
            if (!mp.a_mn) {
                tma_load_2d(sa, tma_a, k0, m0, &full[stage]);
            } else {
#pragma unroll
                for (int b = 0; b < BM / 64; ++b) tma_load_2d(sa + b * (BK * 128), tma_a, m0 + 64 * b, k0, &full[stage]);
            }
            if (!mp.b_mn) {
                tma_load_2d(sb, tma_b, k0, n0, &full[stage]);
            } else {
#pragma unroll
                for (int b = 0; b < BN / 64; ++b) tma_load_2d(sb + b * (BK * 128), tma_b, n0 + 64 * b, k0, &full[stage]);
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
    }
}

// MMA issuer (one thread): 4 x tcgen05.mma (K=16 each) per k-block into the
// current TMEM accumulator; commits free smem stages and publish finished tiles.
__device__ __forceinline__ void mma_loop(const MainParams& mp, uint32_t tmem_base, uint8_t* sA, uint8_t* sB,
                                         uint64_t* full, uint64_t* empty, uint64_t* tfull, uint64_t* tempty) {
    // kind::f16 instruction descriptor: D f32, A/B bf16, majorness, N>>3, M>>4.
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)mp.a_mn << 15) |
                           ((uint32_t)mp.b_mn << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    // K-major: LBO unused (16), SBO = 8 rows * 128 B; advance 32 B per UMMA_K = 16.
    // MN-major: LBO = next 64-wide MN atom column (BK * 128 B), SBO = 8 K-rows * 128 B;
    //           advance 2 x 1024 B per UMMA_K = 16.
    const uint32_t a_lbo = mp.a_mn ? BK * 128 : 16, b_lbo = mp.b_mn ? BK * 128 : 16;
    const uint32_t a_step = mp.a_mn ? 2048 : 32, b_step = mp.b_mn ? 2048 : 32;
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < mp.ntiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < mp.nk; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(sA + stage * A_STAGE_BYTES);
            const uint32_t sb = smem_u32(sB + stage * B_STAGE_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
                const uint64_t ad = umma_desc_sw128(sa + k * a_step, a_lbo, 1024);
                const uint64_t bd = umma_desc_sw128(sb + k * b_step, b_lbo, 1024);
                umma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0);
            }
            umma_commit(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
    }
}

}  // namespace coda
