// coda_fast.cuh — compile-time specialised epilogues for the fused CODA launches.
//
// The generic interpreter (coda_gemm.cuh) executes any valid EpilogueProgram.
// The reference's hot programs (tilefuse/kernels.py:243-557: K1, K2, K4-K7,
// K9, K10 and the plain dgrad/wgrad GEMMs) are additionally compiled as
// flag-specialised kernels with:
//
//   * 8 epilogue warps: warp w reads TMEM lane quadrant w%4 (32 rows, thread ==
//     row) and one 128-column half of the 128x256 accumulator, in 32-column
//     chunks (tcgen05.ld.32x32b.x32);
//   * stores staged through a per-warp 4 KiB swizzled smem buffer and written
//     by TMA (cp.async.bulk.tensor ... bulk_group) — fully coalesced, and the
//     tensor maps clip ragged edges;
//   * thread-local row reductions (sum of squares, <preact, grad>) and a
//     warp-butterfly column reduction (31 shuffles for 32 columns) combined
//     across the four row quadrants through 2 KiB of smem, in fixed order.
//
// Op order is the canonical order of the reference programs:
//   acc_in -> PartialRowDot -> RowScale -> ResidualAdd -> AuxTileStore -> PartialSumSq ->
//   RowVecMul -> PairwiseRope -> PairwiseSwiglu | PairwiseSwigluBackward |
//   RmsNormBackwardLocal -> main store.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include "coda_gemm.cuh"
#include "coda_mainloop.cuh"
#include "coda_ptx.cuh"

namespace coda {

enum FastFlags : int {
    F_ROWSCALE = 1 << 0,
    F_RESIDUAL = 1 << 1,
    F_AUX = 1 << 2,         // AuxTileStore of the running tile (factor 1)
    F_SUMSQ = 1 << 3,
    F_ROWVEC = 1 << 4,
    F_ROPE = 1 << 5,
    F_SWIGLU = 1 << 6,
    F_SWIGLU_BWD = 1 << 7,  // aux = recompute, rowpart = <preact, grad> at factor 2
    F_RMSBWD = 1 << 8,      // aux = normed, colpart = gamma-grad pieces
    F_RMSBWD_ACC = 1 << 9,
    F_STORE_MAIN = 1 << 10,
    F_OUT_F32 = 1 << 11,
    F_GATHER = 1 << 12,     // TargetGather: target[row] = tile[row, label[row]]
    F_LSE = 1 << 13,        // OnlineLse: (max, scaled sum) pairs per piece (rowpart holds pairs)
    F_ROWDOT = 1 << 14,     // PartialRowDot against a side tile, before RowScale (rowpart = row sums)
    F_XENT_BWD = 1 << 15,   // CrossEntropyBackward: grad = (exp(x - lse) - onehot) * scale, rowpart = sum x*grad
    F_PEER = 1 << 16,       // data-parallel weight gradient: cross-rank sum over peer memory (no main store)
};

constexpr int MAX_PEERS = 8;

constexpr int FAST_EPI_WARPS = 8;
constexpr int FAST_THREADS = 64 + 32 * FAST_EPI_WARPS;
constexpr int STG_BYTES = 4096;                   // per epilogue warp: two 2 KiB regions
constexpr int COLRED_BYTES = 2 * 2 * 4 * 32 * 4;  // [half][buf][quadrant][32] f32

struct FastParams {
    MainParams mp;
    const float* acc_in;
    int64_t ld_acc;
    const float* rowscale;
    const void* residual;
    int64_t ld_res;
    const float* rowvec;
    const void* cosp;
    int64_t ld_cos;
    const void* sinp;
    int64_t ld_sin;
    float rope_sign;
    const void* preact2;
    int64_t ld_pre2;
    const void* pre;
    int64_t ld_pre;
    const float* inv_rms;
    const float* gamma;
    const float* stat;
    const void* grad_in;
    int64_t ld_gin;
    float* rowpart;
    int64_t ld_rowpart;
    const int32_t* rowpart_map;
    float* colpart;
    int64_t ld_colpart;
    const int32_t* colpart_map;
    const void* rowdot_x;   // F_ROWDOT: the tile operand X of sum(tile * X)
    int64_t ld_rowdot_x;
    const int64_t* labels;
    float* target;
    const float* xent_lse;  // F_XENT_BWD: per-row log-sum-exp
    float xent_scale;
    // F_PEER: `peer_world` ranks each run this launch on their own token shard.  Tile t is
    // owned by rank t % world; every rank dumps its f32 partial of t into the owner's
    // landing buffer peer_slots[owner] at slot ((t / world) * world + peer_rank) and
    // arrives on the owner's counter peer_ctr[owner][(t / world) * CG + cta rank]; the
    // last arrival sums the world slots in rank order, rounds to bf16 once and stores the
    // tile into every rank's output peer_out[r] (row stride ld_peer_out).  Pointers are
    // peer-mapped (CUDA IPC / NVLink P2P); counters are zero between launches.
    int peer_world, peer_rank;
    float* peer_slots[MAX_PEERS];
    int* peer_ctr[MAX_PEERS];
    __nv_bfloat16* peer_out[MAX_PEERS];
    int64_t ld_peer_out;
    // tail-split workspace: f32 partial accumulators [tail tile][piece < split][rank][128 x 256]
    // and one arrival counter per (tail tile, rank), zero between launches
    float* ws;
    int* flags;
    int ablate;   // measurement-only ablations (results invalid): 1 = no side loads, 2 = no TMA stores
    int backoff;  // [experiments] epilogue accumulator wait: ns of sleep between polls (0 = plain try_wait loop)
    // staged-store destinations (byte strides): the main output and the AuxTileStore
    void* st_main;
    int64_t st_main_ld, st_main_cols;
    void* st_aux;
    int64_t st_aux_ld, st_aux_cols;
    int st_tma;   // staged boxes leave smem by TMA store instead of the lanes' copy-out (host choice)
    // deferred finalizers (coda_step_t.fin_*): the RowScale vector / the RMSNorm-backward
    // stat computed per row from (M, nb) f32 partials and written back by the tn == 0 tiles
    const float* rs_fin;
    int64_t ld_rs_fin;
    int rs_fin_nb, rs_fin_kind;
    float rs_fin_d, rs_fin_eps;
    const float* st_fin;
    int64_t ld_st_fin;
    int st_fin_nb, st_fin_kind;
    float st_fin_d, st_fin_eps;
    // compact RoPE tables (F_ROPE): 0 = full (M, N) cos/sin tables.  h > 0: tma_s0/s1 map
    // (M, h/2) tables of one angle per pair; columns [0, 2h) rotate by pair (col mod h)/2
    // (the q and k spans of the packed projection share angles), columns >= 2h are the
    // identity (cos 1, sin 0) and load nothing.
    int rope_h;
};

// Whole tiles run the program in the unit that computed them; the pieces of a split
// tail tile are reduced by whichever piece finishes last (see the piece path below),
// which is only known at run time, so only whole tiles prefetch their side operands.
__device__ __forceinline__ bool item_prefetches_side(const Work& w) { return w.piece < 0; }
// Arrival counter of one (tail tile, CTA rank, epilogue warp) region: returns the value
// before this arrival.  Release orders this warp's dumped partial before the increment;
// acquire orders the last arriver's reads of the other pieces after it.
__device__ __forceinline__ int counter_arrive(int* c) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(c) : "memory");
    return old;
}
// The same at system scope, for counters in another GPU's memory (F_PEER).
__device__ __forceinline__ int counter_arrive_sys(int* c) {
    int old;
    asm volatile("atom.add.acq_rel.sys.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(c) : "memory");
    return old;
}

// Side operands (residual, cos/sin, preact, pre_norm/grad_in) are TMA-loaded per
// epilogue warp into a 4 KiB swizzled buffer, one 32-row chunk ahead; kernels that
// have them give up one ring stage for the buffers.
constexpr int F_SIDE = F_RESIDUAL | F_ROPE | F_SWIGLU_BWD | F_RMSBWD | F_ROWDOT;
constexpr int SIDE_BYTES = 4096;

template <int CG, int FL>
struct FastGeom {
    static constexpr bool SIDE = (FL & F_SIDE) != 0;
    static constexpr int NS = Geom<CG>::NSTAGE - (SIDE ? 1 : 0);
    static constexpr int RING = NS * Geom<CG>::STAGE;
    static constexpr int SIDE_TOTAL = SIDE ? FAST_EPI_WARPS * SIDE_BYTES : 0;
    // bytes one chunk's side loads deliver to a warp (32 rows)
    static constexpr int CHUNK_BYTES = (FL & F_SWIGLU_BWD) ? 4096
                                     : (FL & F_ROPE) ? 4096
                                     : (FL & F_RMSBWD) ? ((FL & F_RMSBWD_ACC) ? 4096 : 2048)
                                     : (FL & (F_RESIDUAL | F_ROWDOT)) ? 2048 : 0;
};

// F_PEER epilogue of one tile (see FastParams): dump, arrive on the owner's counter, and
// -- last arrival only -- fold the world partials in rank order and store bf16 everywhere.
// Each epilogue warp owns a 32-row x 128-column region; the dump is lane-contiguous
// (float4 k of lane l at (32 k + l) * 16 B) so every warp access covers four whole lines.
template <int CG>
__device__ __forceinline__ void peer_tile(const FastParams& P, int t, int m0, int n0, int rank, int q, int h,
                                          int ew, int lane, uint32_t tmem_base, int& acc, uint32_t& acc_phase,
                                          uint64_t* tfull, uint64_t* tempty, uint32_t* tmem_slot) {
    const int world = P.peer_world;
    const int own = t % world, j = t / world;
    const int64_t region = (int64_t)(q * 2 + h) * (32 * 128) + lane * 4;
    mbar_wait(&tfull[acc], acc_phase);
    tc_fence_after();
    const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + h * 128);
    float* dst = P.peer_slots[own] + ((int64_t)(j * world + P.peer_rank) * CG + rank) * (BM * BN) + region;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld32(tb + c * 32, v);
#pragma unroll
        for (int e = 0; e < 32; e += 4)
            __stcg(reinterpret_cast<float4*>(dst + (c * 8 + e / 4) * 128), make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]));
    }
    tc_fence_before();
    __threadfence_system();
    __syncwarp();
    if (lane == 0) {
        if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
        else mbar_arrive_leader(&tempty[acc]);
    }
    acc ^= 1;
    if (acc == 0) acc_phase ^= 1;
    named_bar_sync(4, 32 * FAST_EPI_WARPS);          // every region of this CTA is dumped
    if (ew == 0 && lane == 0) {
        int* cnt = P.peer_ctr[own] + j * CG + rank;
        const int old = counter_arrive_sys(cnt);
        if (old == world - 1) *cnt = 0;               // every rank is in: reset for the next launch
        tmem_slot[1] = old == world - 1 ? 1u : 0u;
    }
    named_bar_sync(4, 32 * FAST_EPI_WARPS);
    if (tmem_slot[1] == 0u) return;
    __threadfence_system();
    const int64_t row = (int64_t)m0 + q * 32 + lane;
    const bool row_ok = row < P.mp.M;
    const int N = P.mp.N;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0.0f;
        for (int s = 0; s < world; ++s) {             // rank order: bitwise deterministic
            const float* src = P.peer_slots[own] + ((int64_t)(j * world + s) * CG + rank) * (BM * BN) + region + c * 8 * 128;
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
                const float4 u = __ldcg(reinterpret_cast<const float4*>(src + (e / 4) * 128));
                v[e] += u.x;
                v[e + 1] += u.y;
                v[e + 2] += u.z;
                v[e + 3] += u.w;
            }
        }
        const int gcol = n0 + h * 128 + c * 32;
        if (!row_ok || gcol >= N) continue;
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[e] = pack_bf16x2(v[2 * e], v[2 * e + 1]);
        for (int r = 0; r < world; ++r) {
            __nv_bfloat16* o = P.peer_out[r] + row * P.ld_peer_out + gcol;
            if (gcol + 32 <= N && (P.ld_peer_out & 7) == 0) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    reinterpret_cast<uint4*>(o)[e] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
            } else {
                for (int e = 0; e < 32 && gcol + e < N; ++e) o[e] = __float2bfloat16_rn(v[e]);
            }
        }
    }
}

template <int CG, int FL>
constexpr size_t fast_smem_bytes() {
    using FG = FastGeom<CG, FL>;
    return (size_t)FG::RING + (size_t)FAST_EPI_WARPS * STG_BYTES + FG::SIDE_TOTAL + COLRED_BYTES +
           (2 * FG::NS + 4 + FAST_EPI_WARPS) * 8 + 16;
}

// One thread's row of a 32-row side box: RB bytes (64: SWIZZLE_64B, 128: SWIZZLE_128B) of bf16.
template <int RB>
__device__ __forceinline__ void side_row(uint32_t base, int r, float* out) {
    constexpr uint32_t MASK = RB == 128 ? 0x70u : 0x30u;
#pragma unroll
    for (int c = 0; c < RB / 16; ++c) {
        const uint32_t off = (uint32_t)(r * RB + c * 16);
        uint32_t w[4];
        ld_shared_v4(base + (off ^ ((off >> 3) & MASK)), w[0], w[1], w[2], w[3]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            out[c * 8 + 2 * i] = __uint_as_float(w[i] << 16);
            out[c * 8 + 2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
}

// One thread's row of a compact RoPE box (32 rows x 16 bf16, SWIZZLE_32B): 16 angles,
// each duplicated for the two columns of its pair -> 32 values.
__device__ __forceinline__ void side_row_pairs(uint32_t base, int r, float* out) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const uint32_t off = (uint32_t)(r * 32 + c * 16);
        uint32_t w[4];
        ld_shared_v4(base + (off ^ ((off >> 3) & 0x10u)), w[0], w[1], w[2], w[3]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xFFFF0000u);
            out[c * 16 + 4 * i] = lo;
            out[c * 16 + 4 * i + 1] = lo;
            out[c * 16 + 4 * i + 2] = hi;
            out[c * 16 + 4 * i + 3] = hi;
        }
    }
}

// -------------------------------------------------------------- row-segment loads
// W values of a row starting at column c0 into d[]; zero for !ok rows and for
// columns >= ncols (tensor rows are padded to 16 B so a vector that starts
// inside the row never leaves the allocation).
template <typename TS, int W>
__device__ __forceinline__ void fload(const TS* rowp, int64_t c0, int64_t ncols, bool ok, float* d) {
    constexpr int V = Io<TS>::V;
#pragma unroll
    for (int i = 0; i < W; i += V) {
        if (ok && c0 + i < ncols) {
            Io<TS>::load(rowp + c0 + i, d + i);
        } else {
#pragma unroll
            for (int e = 0; e < V; ++e) d[i + e] = 0.0f;
        }
    }
    if (c0 + W > ncols) {
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (c0 + i >= ncols) d[i] = 0.0f;
    }
}

template <int W>
__device__ __forceinline__ void fload_vec(const float* vp, int64_t c0, int64_t n, float* d) {
#pragma unroll
    for (int i = 0; i < W; i += 4) {
        if (c0 + i + 4 <= n) {
            const float4 u = __ldg(reinterpret_cast<const float4*>(vp + c0 + i));
            d[i] = u.x; d[i + 1] = u.y; d[i + 2] = u.z; d[i + 3] = u.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) d[i + e] = (c0 + i + e < n) ? __ldg(vp + c0 + i + e) : 0.0f;
        }
    }
}

template <int W>
__device__ __forceinline__ void fload_vec_cg(const float* vp, int64_t c0, int64_t n, float* d) {
#pragma unroll
    for (int i = 0; i < W; i += 4) {
        if (c0 + i + 4 <= n) {
            const float4 u = __ldcg(reinterpret_cast<const float4*>(vp + c0 + i));
            d[i] = u.x; d[i + 1] = u.y; d[i + 2] = u.z; d[i + 3] = u.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) d[i + e] = (c0 + i + e < n) ? __ldcg(vp + c0 + i + e) : 0.0f;
        }
    }
}

// -------------------------------------------------------------- staged stores
// Thread == row in registers; global rows want whole lines.  Each warp transposes a
// 32 x RB-byte box (RB <= 64) through its own 2 KiB smem region (regions 0 / 1 used
// alternately), then its lanes copy the box out row-contiguously with coalesced 16-B
// global stores: a warp instruction covers 8 rows x 64 B, every 32-B sector whole.
// 128-byte rows (64 bf16 / 32 f32 values) go out as two 64-byte-wide halves.
//
// Round 2 handed each box to the TMA engine (cp.async.bulk.tensor store), which also
// issues the mainloop's operand loads, and every launch ended draining its stores.
// The coalesced copy-out is bit-identical; launched one at a time (per-launch CUDA
// events) K10 (1.41 GB of output) drops 1.70 -> 1.62 ms, K6 -1.3 %, the sum of the C4
// launches -4 %; in the PDL-chained step most of that was already hidden and the step
// gains 0.7-1.2 % (profiles/r02_session3/stdirect_ab.txt, ab_store_path_c4_interleaved.jsonl).
// The TMA path stays for the one launch where the lanes' copy-out costs more than it
// saves: the width-doubling SwiGLU backward (three boxes per chunk) on a short mainloop
// (K < 4096: C3's K10 0.274 ms with TMA stores vs 0.296 ms, profiles/r02_session3/
// ablate_sttma_c3.txt); the host sets FastParams::st_tma (option "st_tma" forces it).
struct Stager {
    uint32_t base;      // smem address of this warp's 4 KiB buffer (1024-aligned)
    int region;
    bool skip;          // ablation: stage into smem but store nothing
    bool tma;           // boxes leave smem by TMA store (FastParams::st_tma)
};

// AUX: the destination is the AuxTileStore output (P.st_aux), else the main output; its
// pointer / strides are read from the kernel parameters at the copy-out (no registers
// held across the epilogue).
// Step 1 of a staged store: this thread's row of a 32 x RB box (RB <= 64) into the
// warp's current region, in the swizzled layout.  Returns the region's smem address.
template <typename TO, int RB>
__device__ __forceinline__ uint32_t stage_box(Stager& sg, const float* v, int lane) {
    constexpr uint32_t MASK = RB == 64 ? 0x30u : 0x10u;
    // TMA path: the region we are about to overwrite was read by the store before last
    if (sg.tma && lane == 0) bulk_wait_read<1>();
    // every lane's copy-out reads of this region (two boxes ago) are done
    __syncwarp();
    const uint32_t rbase = sg.base + (uint32_t)(sg.region * 2048);
#pragma unroll
    for (int c = 0; c < RB / 16; ++c) {
        const uint32_t off = (uint32_t)(lane * RB + c * 16);
        const uint32_t phys = off ^ ((off >> 3) & MASK);
        uint32_t w0, w1, w2, w3;
        if constexpr (sizeof(TO) == 2) {
            w0 = pack_bf16x2(v[c * 8 + 0], v[c * 8 + 1]);
            w1 = pack_bf16x2(v[c * 8 + 2], v[c * 8 + 3]);
            w2 = pack_bf16x2(v[c * 8 + 4], v[c * 8 + 5]);
            w3 = pack_bf16x2(v[c * 8 + 6], v[c * 8 + 7]);
        } else {
            w0 = __float_as_uint(v[c * 4 + 0]);
            w1 = __float_as_uint(v[c * 4 + 1]);
            w2 = __float_as_uint(v[c * 4 + 2]);
            w3 = __float_as_uint(v[c * 4 + 3]);
        }
        st_shared_v4(rbase + phys, w0, w1, w2, w3);
    }
    sg.region ^= 1;
    return rbase;
}

// Step 2: the box at `rbase` (staged by every lane, after a __syncwarp) to global rows
// y.. and byte column x * sizeof(TO).. of the main (AUX = false) or aux output: lane l
// takes 16-B chunks l, l + 32, ... in row-major order.  Pointers and strides are read
// from the kernel parameters here, so nothing is held in registers across the epilogue.
template <typename TO, int RB, bool AUX>
__device__ __forceinline__ void copy_box(const Stager& sg, const FastParams& P, uint32_t rbase, int x, int y,
                                         int lane) {
    constexpr uint32_t MASK = RB == 64 ? 0x30u : 0x10u;
    constexpr int CPR = RB / 16;    // chunks per row
    const int64_t ld = AUX ? P.st_aux_ld : P.st_main_ld;
    const int64_t left = (AUX ? P.st_aux_cols : P.st_main_cols) - (int64_t)x * (int64_t)sizeof(TO);
    const int rows_left = sg.skip ? 0 : P.mp.M - y;
    char* const box = static_cast<char*>(AUX ? P.st_aux : P.st_main) + (int64_t)y * ld +
                      (int64_t)x * (int64_t)sizeof(TO);
    // one 16-B chunk in flight per lane (keeps the register-heavy epilogues spill-free)
#pragma unroll 1
    for (int i = 0; i < CPR; ++i) {
        const int j = i * 32 + lane;
        const int row = j / CPR, c = j % CPR;
        const uint32_t off = (uint32_t)(row * RB + c * 16);
        const uint32_t phys = off ^ ((off >> 3) & MASK);
        uint32_t w[4];
        ld_shared_v4(rbase + phys, w[0], w[1], w[2], w[3]);
        const int64_t rem = left - c * 16;
        if (row >= rows_left || rem <= 0) continue;
        char* p = box + row * ld + c * 16;
        if (rem >= 16) {
            *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
            // ragged last columns: element by element, re-read from smem (no register array)
#pragma unroll 1
            for (int k = 0; k < (int)rem; k += (int)sizeof(TO)) {
                if constexpr (sizeof(TO) == 4) {
                    uint32_t e;
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(e) : "r"(rbase + phys + k));
                    *reinterpret_cast<uint32_t*>(p + k) = e;
                } else {
                    unsigned short e;
                    asm volatile("ld.shared.b16 %0, [%1];" : "=h"(e) : "r"(rbase + phys + k));
                    *reinterpret_cast<unsigned short*>(p + k) = e;
                }
            }
        }
    }
}

// A whole staged store of W values per row: stage, then copy out (or, experiment
// st_tma, hand the box to the TMA engine).
template <typename TO, int W, bool AUX = false>
__device__ __forceinline__ void staged_store(Stager& sg, const FastParams& P, const CUtensorMap* tm, int x, int y,
                                             const float* v, int lane) {
    constexpr int RB = W * (int)sizeof(TO);
    static_assert(RB == 32 || RB == 64 || RB == 128, "row bytes per staged store");
    if constexpr (RB == 128) {
        // (TMA maps of 128-byte rows have a W/2-column box: host make_map)
        staged_store<TO, W / 2, AUX>(sg, P, tm, x, y, v, lane);
        staged_store<TO, W / 2, AUX>(sg, P, tm, x + W / 2, y, v + W / 2, lane);
    } else {
        const uint32_t rbase = stage_box<TO, RB>(sg, v, lane);
        if (sg.tma) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && !sg.skip) {
                tma_store_2d(tm, rbase, x, y);
                bulk_commit();
            }
            return;
        }
        __syncwarp();
        copy_box<TO, RB, AUX>(sg, P, rbase, x, y, lane);
    }
}

// Deferred form for register-heavy epilogues: stage now (registers -> smem), copy out
// later with copy_box when fewer values are live.  At most one deferred box may be
// pending when the next box is staged (two regions).
template <typename TO, int W>
__device__ __forceinline__ void staged_defer(Stager& sg, const float* v, int lane) {
    static_assert(W * (int)sizeof(TO) <= 64, "deferred boxes are at most 64 bytes per row");
    stage_box<TO, W * (int)sizeof(TO)>(sg, v, lane);
}

// Column sums over the warp's 32 rows: lane l ends with column l (fixed tree).
__device__ __forceinline__ float warp_colsum32(float (&x)[32], int lane) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
            const float send = up ? x[i] : x[i + off];
            const float keep = up ? x[i + off] : x[i];
            x[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return x[0];
}

// -------------------------------------------------------------- kernel
template <typename TS, int FL, int CG>
__global__ void __launch_bounds__(FAST_THREADS, 1)
coda_gemm_fast(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
               const __grid_constant__ CUtensorMap tma_main, const __grid_constant__ CUtensorMap tma_aux,
               const __grid_constant__ CUtensorMap tma_s0, const __grid_constant__ CUtensorMap tma_s1,
               const __grid_constant__ FastParams P) {
    using G = Geom<CG>;
    using FG = FastGeom<CG, FL>;
    constexpr int NS = FG::NS;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + NS * G::A_BYTES;
    uint8_t* stg = smem + FG::RING;
    uint8_t* side = stg + FAST_EPI_WARPS * STG_BYTES;
    float* colred = reinterpret_cast<float*>(side + FG::SIDE_TOTAL);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(colred) + COLRED_BYTES);
    uint64_t* empty = full + NS;
    uint64_t* tfull = empty + NS;
    uint64_t* tempty = tfull + 2;
    uint64_t* sidebar = tempty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sidebar + FAST_EPI_WARPS);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const MainParams& mp = P.mp;
    const int rank = CG == 1 ? 0 : (int)cluster_ctarank();
    const int unit = CG == 1 ? (int)blockIdx.x : (int)cluster_id_x();
    const int nunits = CG == 1 ? (int)gridDim.x : (int)nclusters_x();

    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023u) __trap();   // swizzled TMA buffers need 1 KiB alignment
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], FAST_EPI_WARPS * CG);   // one arrival per epilogue warp of the pair
        }
        for (int s = 0; s < FAST_EPI_WARPS; ++s) mbar_init(&sidebar[s], 1);
        fence_mbar_init();
        tma_prefetch_desc(&tma_a);
        tma_prefetch_desc(&tma_b);
        if (FL & F_STORE_MAIN) tma_prefetch_desc(&tma_main);
        if (FL & (F_AUX | F_SWIGLU_BWD | F_RMSBWD)) tma_prefetch_desc(&tma_aux);
        if (FG::SIDE) {
            tma_prefetch_desc(&tma_s0);
            if (FL & (F_ROPE | F_RMSBWD_ACC)) tma_prefetch_desc(&tma_s1);
        }
    }
    if (warp == 1) {
        if constexpr (CG == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
        else tmem_alloc_pair<TMEM_COLS>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();   // peer barriers initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // PDL: let the next launch start its prologue, and wait for the previous one's
    // results before any global-memory access.
    griddep_launch_dependents();
    griddep_wait();

    if (warp == 0) {
        producer_loop<CG, NS>(mp, &tma_a, &tma_b, sA, sB, full, empty, rank, unit, nunits);
    } else if (warp == 1) {
        if (rank == 0) mma_loop<CG, NS>(mp, tmem_base, sA, sB, full, empty, tfull, tempty, unit, nunits);
    } else {
        const int ew = warp - 2;            // 0..7
        const int q = warp & 3;             // TMEM lane quadrant
        const int h = ew >> 2;              // column half of the 256-wide tile
        const int lrow = q * 32 + lane;
        const int M = mp.M, N = mp.N;
        Stager sg{smem_u32(stg + ew * STG_BYTES), 0, (P.ablate & 2) != 0, P.st_tma != 0};
        int cbuf = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        const uint32_t sbase = smem_u32(side + ew * SIDE_BYTES);
        uint32_t side_phase = 0;
        // lane 0: TMA-load the side operands of chunk c of tile t into this warp's buffer
        const bool no_side = (P.ablate & 1) != 0;
        const int rope_h = (FL & F_ROPE) ? P.rope_h : 0;
        // does the chunk starting at global column x load side operands?  (issue and wait
        // sides evaluate the same predicate)
        auto side_needed = [&](int x) { return !no_side && !(rope_h > 0 && x >= 2 * rope_h); };
        auto side_issue = [&](int tm_, int tn_, int c_) {
            const int y = tm_ * G::TILE_M + rank * BM + q * 32;
            const int x = tn_ * BN + h * 128 + c_ * 32;
            if (!side_needed(x)) return;
            fence_proxy_async_smem();
            if ((FL & F_ROPE) && rope_h > 0) {
                // one angle per pair: 16 columns (32 B) of each compact table
                const int pc = (x % (rope_h > 0 ? rope_h : 1)) / 2;
                mbar_arrive_expect_tx(&sidebar[ew], 2048);
                tma_load_2d(sbase, &tma_s0, pc, y, &sidebar[ew]);
                tma_load_2d(sbase + 2048, &tma_s1, pc, y, &sidebar[ew]);
                return;
            }
            mbar_arrive_expect_tx(&sidebar[ew], FG::CHUNK_BYTES);
            if (FL & F_SWIGLU_BWD) {
                tma_load_2d(sbase, &tma_s0, 2 * x, y, &sidebar[ew]);
            } else {
                tma_load_2d(sbase, &tma_s0, x, y, &sidebar[ew]);
                if (FL & (F_ROPE | F_RMSBWD_ACC)) tma_load_2d(sbase + 2048, &tma_s1, x, y, &sidebar[ew]);
            }
        };
        if (FG::SIDE && lane == 0 && unit < mp.nitems) {
            const Work w0 = work_item(mp, unit);
            if (item_prefetches_side(w0)) side_issue(w0.tm, w0.tn, 0);
        }
        const int split = mp.split;
        for (int i = unit; i < mp.nitems; i += nunits) {
            const Work w = work_item(mp, i);
            const int tm = w.tm, tn = w.tn;
            const int m0 = tm * G::TILE_M + rank * BM;
            const int n0 = tn * BN;
            if constexpr ((FL & F_PEER) != 0) {
                peer_tile<CG>(P, tm * mp.ntn + tn, m0, n0, rank, q, h, ew, lane, tmem_base, acc, acc_phase, tfull, tempty,
                          tmem_slot);
                continue;
            }
            // a K piece of a split tail tile: every epilogue warp dumps the raw f32 accumulator
            // of its 32 x 128 region; then the CTA arrives once on the (tail tile, rank) counter.
            // The last of the `split` arrivals sums every dumped piece in fixed piece order and
            // runs the program; the others are done.  No piece ever waits for another, so the
            // launch needs no co-residency of its clusters.  The decision is per CTA (not per
            // warp) because the program's column reductions synchronise the warps of a half.
            const bool piece = w.piece >= 0;
            // dump layout of a warp's 32 x 128 region: float4 k of lane l at (k * 32 + l) * 4,
            // so every warp-wide store / load covers 512 contiguous bytes (4 full lines)
            const int64_t ws_region = (int64_t)(q * 2 + h) * (32 * 128) + lane * 4;
            if (piece) {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + h * 128);
                float* dst = P.ws + ((int64_t)(w.tail_idx * split + w.piece) * CG + rank) * (BM * BN) + ws_region;
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    float v[32];
                    tmem_ld32(tb + c * 32, v);
#pragma unroll
                    for (int e = 0; e < 32; e += 4)
                        __stcg(reinterpret_cast<float4*>(dst + (c * 8 + e / 4) * 128),
                               make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]));
                }
                tc_fence_before();
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
                    else mbar_arrive_leader(&tempty[acc]);
                }
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
                named_bar_sync(4, 32 * FAST_EPI_WARPS);          // every region of this CTA is dumped
                if (ew == 0 && lane == 0) {
                    int* cnt = P.flags + w.tail_idx * CG + rank;
                    const int old = counter_arrive(cnt);
                    if (old == split - 1) *cnt = 0;               // every arrival is in: reset
                    tmem_slot[1] = old == split - 1 ? 1u : 0u;
                }
                named_bar_sync(4, 32 * FAST_EPI_WARPS);
                if (tmem_slot[1] == 0u) continue;
                __threadfence();
                if (FG::SIDE && lane == 0) side_issue(tm, tn, 0);
            }
            const int64_t row = (int64_t)m0 + lrow;
            const bool row_ok = row < M;
            float rsc = 1.0f, rr = 0.0f, ss = 0.0f;
            if ((FL & F_ROWSCALE) && row_ok) {
                if (P.rs_fin != nullptr) {
                    rsc = finalize_row(P.rs_fin + row * P.ld_rs_fin, P.rs_fin_nb, P.rs_fin_kind, P.rs_fin_d,
                                       P.rs_fin_eps);
                    if (tn == 0 && h == 0) const_cast<float*>(P.rowscale)[row] = rsc;
                } else {
                    rsc = __ldg(P.rowscale + row);
                }
            }
            if ((FL & F_RMSBWD) && row_ok) {
                rr = __ldg(P.inv_rms + row);
                if (P.st_fin != nullptr) {
                    ss = finalize_row(P.st_fin + row * P.ld_st_fin, P.st_fin_nb, P.st_fin_kind, P.st_fin_d,
                                      P.st_fin_eps);
                    if (tn == 0 && h == 0) const_cast<float*>(P.stat)[row] = ss;
                } else {
                    ss = __ldg(P.stat + row);
                }
            }
            float pacc = 0.0f, pmax = -INFINITY;
            int ppid = -1;
            int64_t label = -1;
            if ((FL & (F_GATHER | F_XENT_BWD)) && row_ok) label = __ldg(P.labels + row);
            float xlse = 0.0f;
            if ((FL & F_XENT_BWD) && row_ok) xlse = __ldg(P.xent_lse + row);

            // CTA-scope wait: the accumulator is read through tcgen05.ld after the fence below;
            // a cluster-scope acquire would emit an L1 invalidate (CCTL.IVALL) on every poll.
            if (!piece) {
#ifdef CODA_EXPERIMENTS
                if (P.backoff > 0) mbar_wait_backoff(&tfull[acc], acc_phase, P.backoff);
                else
#endif
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
            }
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + h * 128);

#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                float v[32];
                if (!piece) {
                    tmem_ld32(tbase + c * 32, v);
                    if (c == 3) {
                        // this warp's share of the accumulator is in registers: release it
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
                            else mbar_arrive_leader(&tempty[acc]);
                        }
                    }
                } else {
                    // fixed-order sum of every K piece (L2 loads, bypassing L1)
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.0f;
                    for (int pc = 0; pc < split; ++pc) {
                        const float* src = P.ws + ((int64_t)(w.tail_idx * split + pc) * CG + rank) * (BM * BN) +
                                           ws_region + c * 8 * 128;
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const float4 u = __ldcg(reinterpret_cast<const float4*>(src + (e / 4) * 128));
                            v[e] += u.x;
                            v[e + 1] += u.y;
                            v[e + 2] += u.z;
                            v[e + 3] += u.w;
                        }
                    }
                }
                // side operands of this chunk: wait for the TMA load, pull this thread's row
                // into registers, then reuse the buffer for the next chunk's load
                float sd0[FG::SIDE ? ((FL & F_SWIGLU_BWD) ? 64 : 32) : 1];
                float sd1[(FL & (F_ROPE | F_RMSBWD_ACC)) ? 32 : 1];
                if constexpr (FG::SIDE) {
                    const int xcol = n0 + h * 128 + c * 32;
                    const bool loaded = side_needed(xcol);
                    if (loaded) {
                        mbar_wait(&sidebar[ew], side_phase);
                        side_phase ^= 1;
                    }
                    if constexpr ((FL & F_ROPE) != 0) {
                        if (rope_h > 0) {
                            if (loaded) {
                                side_row_pairs(sbase, lane, sd0);
                                side_row_pairs(sbase + 2048, lane, sd1);
                            } else {
#pragma unroll
                                for (int e = 0; e < 32; ++e) {
                                    sd0[e] = 1.0f;
                                    sd1[e] = 0.0f;
                                }
                            }
                        } else {
                            side_row<64>(sbase, lane, sd0);
                            side_row<64>(sbase + 2048, lane, sd1);
                        }
                    } else {
                        if constexpr ((FL & F_SWIGLU_BWD) != 0) side_row<128>(sbase, lane, sd0);
                        else side_row<64>(sbase, lane, sd0);
                        if constexpr ((FL & F_RMSBWD_ACC) != 0) side_row<64>(sbase + 2048, lane, sd1);
                    }
                    __syncwarp();
                    if (lane == 0) {
                        if (c < 3) {
                            side_issue(tm, tn, c + 1);
                        } else if (i + nunits < mp.nitems) {
                            const Work wn = work_item(mp, i + nunits);
                            if (item_prefetches_side(wn)) side_issue(wn.tm, wn.tn, 0);
                        }
                    }
                }
                const int gcol0 = n0 + h * 128 + c * 32;
                if (gcol0 >= N) continue;   // uniform for the 4 warps of this half
                const bool edge = gcol0 + 32 > N;
                if (P.acc_in != nullptr) {
                    float x[32];
                    fload<float, 32>(P.acc_in + row * P.ld_acc, gcol0, N, row_ok, x);
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] += x[i];
                }
                if constexpr ((FL & F_ROWDOT) != 0) {
                    // PartialRowDot(X) ahead of RowScale: sum(tile * X) of this row's piece
                    float s = 0.0f;
#pragma unroll
                    for (int i = 0; i < 32; ++i) s += v[i] * sd0[i];
                    const int pid = __ldg(P.rowpart_map + gcol0);
                    if (pid != ppid) {
                        if (ppid >= 0 && row_ok) P.rowpart[row * P.ld_rowpart + ppid] = pacc;
                        ppid = pid;
                        pacc = 0.0f;
                    }
                    pacc += s;
                }
                if (FL & F_ROWSCALE) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] *= rsc;
                }
                if constexpr ((FL & F_RESIDUAL) != 0) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] += sd0[i];
                }
                if (FL & F_AUX) staged_store<TS, 32, true>(sg, P, &tma_aux, gcol0, m0 + q * 32, v, lane);
                if (FL & F_SUMSQ) {
                    float s = 0.0f;
#pragma unroll
                    for (int i = 0; i < 32; ++i) s += v[i] * v[i];
                    const int pid = __ldg(P.rowpart_map + gcol0);
                    if (pid != ppid) {
                        if (ppid >= 0 && row_ok) P.rowpart[row * P.ld_rowpart + ppid] = pacc;
                        ppid = pid;
                        pacc = 0.0f;
                    }
                    pacc += s;
                }
                if (FL & F_ROWVEC) {
                    float g[32];
                    fload_vec<32>(P.rowvec, gcol0, N, g);
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] *= g[i];
                }
                if constexpr ((FL & F_ROPE) != 0) {
                    const float* cs = sd0;
                    const float* sn = sd1;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float x0 = v[2 * k], x1 = v[2 * k + 1];
                        const float se = P.rope_sign * sn[2 * k], so = P.rope_sign * sn[2 * k + 1];
                        v[2 * k] = x0 * cs[2 * k] - x1 * se;
                        v[2 * k + 1] = x0 * so + x1 * cs[2 * k + 1];
                    }
                }
                if (FL & F_GATHER) {
                    const int64_t local = label - gcol0;
                    if (local >= 0 && local < 32 && label < N) {
                        // select v[local] with a 5-level select tree over the bits of local:
                        // static register indices only (a dynamic v[local] would put the
                        // whole chunk in local memory every chunk)
                        const int l = (int)local;
                        float t16[16], t8[8], t4[4], t2[2];
#pragma unroll
                        for (int i = 0; i < 16; ++i) t16[i] = (l & 16) ? v[i + 16] : v[i];
#pragma unroll
                        for (int i = 0; i < 8; ++i) t8[i] = (l & 8) ? t16[i + 8] : t16[i];
#pragma unroll
                        for (int i = 0; i < 4; ++i) t4[i] = (l & 4) ? t8[i + 4] : t8[i];
#pragma unroll
                        for (int i = 0; i < 2; ++i) t2[i] = (l & 2) ? t4[i + 2] : t4[i];
                        P.target[row] = (l & 1) ? t2[1] : t2[0];
                    }
                }
                if (FL & F_LSE) {
                    // chunk-level (max, sum exp) merged into the running pair of this piece
                    float mc = -INFINITY;
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (!edge || gcol0 + i < N) mc = fmaxf(mc, v[i]);
                    float sc = 0.0f;
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (!edge || gcol0 + i < N) sc += __expf(v[i] - mc);
                    const int pid = __ldg(P.rowpart_map + gcol0);
                    if (pid != ppid) {
                        if (ppid >= 0 && row_ok) {
                            P.rowpart[row * P.ld_rowpart + 2 * ppid] = pmax;
                            P.rowpart[row * P.ld_rowpart + 2 * ppid + 1] = pacc;
                        }
                        ppid = pid;
                        pacc = 0.0f;
                        pmax = -INFINITY;
                    }
                    const float mn = fmaxf(pmax, mc);
                    pacc = pacc * (pmax == -INFINITY ? 0.0f : __expf(pmax - mn)) + sc * __expf(mc - mn);
                    pmax = mn;
                }
                if constexpr ((FL & F_XENT_BWD) != 0) {
                    float s = 0.0f;
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        float pr = __expf(v[i] - xlse);
                        if (gcol0 + i == label) pr -= 1.0f;
                        pr *= P.xent_scale;
                        if (!edge || gcol0 + i < N) s += v[i] * pr;
                        v[i] = pr;
                    }
                    const int pid = __ldg(P.rowpart_map + gcol0);
                    if (pid != ppid) {
                        if (ppid >= 0 && row_ok) P.rowpart[row * P.ld_rowpart + ppid] = pacc;
                        ppid = pid;
                        pacc = 0.0f;
                    }
                    pacc += s;
                }
                if (FL & F_SWIGLU) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float g = v[2 * k], u = v[2 * k + 1];
                        v[k] = g * sigmoid_stable(g) * u;
                    }
                    if (FL & F_STORE_MAIN) staged_store<TS, 16>(sg, P, &tma_main, gcol0 / 2, m0 + q * 32, v, lane);
                } else if (FL & F_SWIGLU_BWD) {
                    const float* z = sd0;
                    float rec[32];
                    float s = 0.0f;
                    float o[64];
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        const float g = z[2 * k], u = z[2 * k + 1], dd = v[k];
                        const float sg_ = sigmoid_stable(g);
                        const float sl = g * sg_;
                        rec[k] = sl * u;
                        const float gu = dd * sl;
                        const float gg = dd * u * (sg_ + sl * (1.0f - sg_));
                        o[2 * k] = gg;
                        o[2 * k + 1] = gu;
                        s += g * gg;
                        s += u * gu;
                    }
                    staged_store<TS, 32, true>(sg, P, &tma_aux, gcol0, m0 + q * 32, rec, lane);
                    const int pid = __ldg(P.rowpart_map + 2 * gcol0);
                    if (pid != ppid) {
                        if (ppid >= 0 && row_ok) P.rowpart[row * P.ld_rowpart + ppid] = pacc;
                        ppid = pid;
                        pacc = 0.0f;
                    }
                    pacc += s;
                    if (FL & F_STORE_MAIN) staged_store<TS, 64>(sg, P, &tma_main, 2 * gcol0, m0 + q * 32, o, lane);
                } else if (FL & F_RMSBWD) {
                    float g[32], tmp[32];
                    float* cp = sd0;
                    {
                        float g0[32];
                        fload_vec<32>(P.gamma, gcol0, N, g0);
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            cp[i] *= rr;              // c_n
                            tmp[i] = cp[i] * g0[i];   // normed
                        }
                    }
                    // the normed aux box is staged now and copied out after the main store,
                    // when only the outputs are live
                    if (sg.tma) staged_store<TS, 32, true>(sg, P, &tma_aux, gcol0, m0 + q * 32, tmp, lane);
                    else staged_defer<TS, 32>(sg, tmp, lane);
                    // gamma again (L1-resident; an L2-hinted load the compiler does not merge with
                    // the first), so it is not held live across the staging
                    fload_vec_cg<32>(P.gamma, gcol0, N, g);
                    // one pass: the gamma-grad terms D * c_n, and the output (D g - c_n s) r (+ grad_in)
                    // in place -- c_n, g and grad_in die element by element, so the column sum below
                    // runs with only its 32 inputs and the 32 outputs live (no spills at 168 regs)
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        tmp[i] = v[i] * cp[i];
                        v[i] = (v[i] * g[i] - cp[i] * ss) * rr;
                        if constexpr ((FL & F_RMSBWD_ACC) != 0) v[i] += sd1[i];
                    }
                    const float csum = warp_colsum32(tmp, lane);
                    float* red = colred + ((h * 2 + cbuf) * 4) * 32;
                    red[q * 32 + lane] = csum;
                    named_bar_sync(2 + h, 128);
                    if (q == 0) {
                        const int gc = gcol0 + lane;
                        if (gc < N) {
                            int pid = -1;
                            float a = 0.0f;
#pragma unroll
                            for (int qq = 0; qq < 4; ++qq) {
                                const int r0 = m0 + 32 * qq;
                                if (r0 < M) {
                                    const int p = __ldg(P.colpart_map + r0);
                                    if (p != pid) {
                                        if (pid >= 0) P.colpart[(int64_t)pid * P.ld_colpart + gc] = a;
                                        pid = p;
                                        a = 0.0f;
                                    }
                                    a += red[qq * 32 + lane];
                                }
                            }
                            if (pid >= 0) P.colpart[(int64_t)pid * P.ld_colpart + gc] = a;
                        }
                    }
                    cbuf ^= 1;
                    if (FL & F_STORE_MAIN) staged_store<TS, 32>(sg, P, &tma_main, gcol0, m0 + q * 32, v, lane);
                    if (!sg.tma) {
                        // the aux box sits in the region before the current one, or in the one
                        // before that when the main store went between (two regions)
                        const int r = (FL & F_STORE_MAIN) ? sg.region : sg.region ^ 1;
                        __syncwarp();
                        copy_box<TS, 64, true>(sg, P, sg.base + (uint32_t)(r * 2048), gcol0, m0 + q * 32, lane);
                    }
                } else if (FL & F_STORE_MAIN) {
                    if (FL & F_OUT_F32) staged_store<float, 32>(sg, P, &tma_main, gcol0, m0 + q * 32, v, lane);
                    else staged_store<TS, 32>(sg, P, &tma_main, gcol0, m0 + q * 32, v, lane);
                }
            }
            if ((FL & (F_SUMSQ | F_SWIGLU_BWD | F_ROWDOT | F_XENT_BWD)) && ppid >= 0 && row_ok)
                P.rowpart[row * P.ld_rowpart + ppid] = pacc;
            if ((FL & F_LSE) && ppid >= 0 && row_ok) {
                P.rowpart[row * P.ld_rowpart + 2 * ppid] = pmax;
                P.rowpart[row * P.ld_rowpart + 2 * ppid + 1] = pacc;
            }
            if (!piece) {
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
        if (lane == 0) bulk_wait<0>();
        __syncwarp();
    }

    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();   // both CTAs done with the paired TMEM
    if (warp == 1) {
        tc_fence_after();
        if constexpr (CG == 1) tmem_dealloc<TMEM_COLS>(tmem_base);
        else tmem_dealloc_pair<TMEM_COLS>(tmem_base);
    }
}

}  // namespace coda
