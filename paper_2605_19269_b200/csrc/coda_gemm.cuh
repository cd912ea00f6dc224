// coda_gemm.cuh — the fixed GEMM mainloop with a composable epilogue.
//
// One persistent, warp-specialised sm_100a kernel replaces the reference's
// simulated launch `run_gemm` (pkg/src/tilefuse/engine.py:376-464):
//
//   warp 0      TMA producer: 4-stage SWIZZLE_128B smem ring of A/B k-blocks
//   warp 1      MMA issuer:   tcgen05.mma.cta_group::1.kind::f16, 128x256 tile,
//                             f32 accumulator in TMEM, double-buffered (2 x 256 cols)
//   warps 2..5  epilogue:     tcgen05.ld.32x32b -> registers (thread == tile row),
//                             runs the program steps (epilogue.py:606-698) on
//                             32-column chunks, stores with 16-byte vectors,
//                             while the MMA warp runs the next tile's mainloop.
//
// Operand majorness follows the reference's layouts (engine.py:402-403, 436-437):
//   A (m,k) -> K-major,  A (k,m) [trans_a] -> MN-major
//   B (k,n) -> MN-major, B (n,k) [trans_b] -> K-major
// Both are expressed purely through the TMA boxes and UMMA smem descriptors,
// so the same binary serves forward (NN), dgrad (NT) and wgrad (TN).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include "coda_ptx.cuh"
#include "coda_mainloop.cuh"

namespace coda {

constexpr int EPI_WARPS = 4;
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;   // producer, mma, 4 epilogue warps
constexpr int CHUNK = 32;                    // accumulator columns per tcgen05.ld
constexpr int RED_LD = 33;                   // padded row stride of the col-sum scratch

constexpr int MAX_STEPS = 16;
constexpr int MAX_SLOTS = 16;
constexpr int MAX_ROW_STREAMS = 4;           // row-directed partial streams per program

enum OpCode : int {
    OP_ROW_VEC_MUL = 1, OP_ROW_SCALE = 2, OP_RESIDUAL_ADD = 3, OP_AUX_TILE_STORE = 4,
    OP_PARTIAL_SUMSQ = 5, OP_PARTIAL_ROWDOT = 6, OP_PARTIAL_COLSUM = 7, OP_ONLINE_LSE = 8,
    OP_TARGET_GATHER = 9, OP_ROPE = 10, OP_SWIGLU = 11, OP_SWIGLU_BWD = 12, OP_RMSNORM_BWD = 13,
    OP_XENT_BWD = 14,
};

struct DevStep {
    int op;
    int w;          // running width in values per 32-column chunk at step entry (1, 2, 4, ..., 64)
    int a[7];
    int fin_src;    // deferred finalizer: 1 + operand slot of the (m, nb) f32 partials, or 0
    int fin_kind;   // 1 finalize_rms, 2 finalize_rowdot
    int fin_d;
    float fin_eps;
};

// The finalizers of reductions.py:64-98 for one row, in their f32 op order (ascending
// block sum, IEEE-rounded div / sqrt): bit-identical to coda_finalize_rms / _rowdot.
__device__ __forceinline__ float finalize_row(const float* __restrict__ p, int nb, int kind, float d, float eps) {
    float t = 0.0f;
#pragma unroll 8
    for (int b = 0; b < nb; ++b) t = __fadd_rn(t, __ldg(p + b));
    return kind == 1 ? __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(t, d), eps))) : __fdiv_rn(t, d);
}
struct DevOperand {
    const void* ptr;
    int64_t ld;
    int64_t cols;   // logical width (for masking)
};
struct DevStore {
    void* ptr;
    int64_t ld;
    int64_t cols;            // logical width (tile) / piece columns
    const int32_t* map;      // piece map (row-sum: per scaled column, col-sum: per row)
};

struct GemmParams {
    int M, N, K;
    int ntm, ntn, nk, ntiles;
    int a_mn, b_mn;
    int nsteps;
    int store_main, out_f32, out_w;   // out_w: values per chunk at program end
    void* out;
    int64_t ld_out;
    const float* acc_in;     // optional f32 (M, N) added before the program (K-chunked SIM32 GEMMs)
    int64_t ld_acc;
    DevStep steps[MAX_STEPS];
    DevOperand opnd[MAX_SLOTS];
    DevStore store[MAX_SLOTS];
};

// ----------------------------------------------------------------- storage I/O
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename TS> struct Io;

template <> struct Io<__nv_bfloat16> {
    static constexpr int V = 8;
    __device__ static __forceinline__ void load(const __nv_bfloat16* p, float* d) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            d[2 * i] = __uint_as_float(w[i] << 16);
            d[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
    __device__ static __forceinline__ void store(__nv_bfloat16* p, const float* s) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            __nv_bfloat162 h = __floats2bfloat162_rn(s[2 * i], s[2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    __device__ static __forceinline__ void load_shared(const __nv_bfloat16* p, float* d) {
        const uint4 u = *reinterpret_cast<const uint4*>(p);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            d[2 * i] = __uint_as_float(w[i] << 16);
            d[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
    __device__ static __forceinline__ float load1(const __nv_bfloat16* p) { return __bfloat162float(p[0]); }
    __device__ static __forceinline__ void store1(__nv_bfloat16* p, float x) { p[0] = __float2bfloat16_rn(x); }
};

template <> struct Io<float> {
    static constexpr int V = 4;
    __device__ static __forceinline__ void load(const float* p, float* d) {
        const float4 u = __ldg(reinterpret_cast<const float4*>(p));
        d[0] = u.x; d[1] = u.y; d[2] = u.z; d[3] = u.w;
    }
    __device__ static __forceinline__ void store(float* p, const float* s) {
        *reinterpret_cast<float4*>(p) = make_float4(s[0], s[1], s[2], s[3]);
    }
    __device__ static __forceinline__ float load1(const float* p) { return p[0]; }
    __device__ static __forceinline__ void store1(float* p, float x) { p[0] = x; }
};

// Load W values of one row segment [c0, c0+W) (columns >= ncols read as 0).  Segments
// narrower than one 16-byte vector (running width factors below 1/4) go element-wise.
template <typename TS, int W>
__device__ __forceinline__ void load_seg(const TS* rowp, int64_t c0, int64_t ncols, float* d) {
    constexpr int V = Io<TS>::V;
    if constexpr (W < V) {
#pragma unroll
        for (int e = 0; e < W; ++e) d[e] = (c0 + e < ncols) ? Io<TS>::load1(rowp + c0 + e) : 0.0f;
    } else {
#pragma unroll
        for (int i = 0; i < W; i += V) {
            if (c0 + i + V <= ncols) {
                Io<TS>::load(rowp + c0 + i, d + i);
            } else {
#pragma unroll
                for (int e = 0; e < V; ++e)
                    d[i + e] = (c0 + i + e < ncols) ? Io<TS>::load1(rowp + c0 + i + e) : 0.0f;
            }
        }
    }
}
// Store W values (rounded to TS) of one row segment, masking columns >= ncols.
template <typename TS, int W>
__device__ __forceinline__ void store_seg(TS* rowp, int64_t c0, int64_t ncols, const float* s) {
    constexpr int V = Io<TS>::V;
    if constexpr (W < V) {
#pragma unroll
        for (int e = 0; e < W; ++e)
            if (c0 + e < ncols) Io<TS>::store1(rowp + c0 + e, s[e]);
    } else {
#pragma unroll
        for (int i = 0; i < W; i += V) {
            if (c0 + i + V <= ncols) {
                Io<TS>::store(rowp + c0 + i, s + i);
            } else {
#pragma unroll
                for (int e = 0; e < V; ++e)
                    if (c0 + i + e < ncols) Io<TS>::store1(rowp + c0 + i + e, s[i + e]);
            }
        }
    }
}
// Broadcast f32 vector segment (row vector operand, same for all rows).
template <int W>
__device__ __forceinline__ void load_vec_seg(const float* vp, int64_t c0, int64_t n, float* d) {
    if constexpr (W < 4) {
#pragma unroll
        for (int e = 0; e < W; ++e) d[e] = (c0 + e < n) ? __ldg(vp + c0 + e) : 0.0f;
    } else {
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
}

// Run f(Width<W>{}) for the running width w (values per 32-column chunk), so each op body
// is compiled once per width with static register indexing.
template <int W> struct Width { static constexpr int value = W; };
template <typename F>
__device__ __forceinline__ void with_width(int w, F&& f) {
    switch (w) {
    case 1: f(Width<1>{}); break;
    case 2: f(Width<2>{}); break;
    case 4: f(Width<4>{}); break;
    case 8: f(Width<8>{}); break;
    case 16: f(Width<16>{}); break;
    case 32: f(Width<32>{}); break;
    default: f(Width<64>{}); break;
    }
}

// Running row-directed partial (row-sum or (max, sum) pair) of one thread.
struct RowPart {
    float acc;
    float mx;
    int pid;
};

__device__ __forceinline__ void rowpart_flush(const DevStore& st, RowPart& p, int64_t row, bool row_ok,
                                              bool pair) {
    if (row_ok && p.pid >= 0) {
        float* o = static_cast<float*>(st.ptr) + row * st.ld;
        if (pair) {
            o[2 * p.pid] = p.mx;
            o[2 * p.pid + 1] = p.acc;
        } else {
            o[p.pid] = p.acc;
        }
    }
}

// Accumulate W row-sum contributions x[i] at scaled columns c0+i into the
// piece-blocked partial.  Pieces never straddle GPU tiles, so a chunk whose
// first and last valid column share a piece takes the fast path.
template <int W>
__device__ __forceinline__ void rowsum_accum(const DevStore& st, RowPart& p, int64_t row, bool row_ok,
                                             int64_t c0, int64_t ncols, const float* x) {
    const int64_t last = (c0 + W <= ncols ? c0 + W : ncols) - 1;
    if (last < c0) return;
    const int p0 = __ldg(st.map + c0);
    const int p1 = __ldg(st.map + last);
    if (p0 == p1) {
        if (p0 != p.pid) {
            rowpart_flush(st, p, row, row_ok, false);
            p.pid = p0;
            p.acc = 0.0f;
        }
        float s = p.acc;
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (c0 + i <= last) s += x[i];
        p.acc = s;
    } else {
#pragma unroll
        for (int i = 0; i < W; ++i) {
            if (c0 + i <= last) {
                const int q = __ldg(st.map + c0 + i);
                if (q != p.pid) {
                    rowpart_flush(st, p, row, row_ok, false);
                    p.pid = q;
                    p.acc = 0.0f;
                }
                p.acc += x[i];
            }
        }
    }
}

// Online (max, scaled-sum) update in ascending column order (epilogue.py:355-366).
template <int W>
__device__ __forceinline__ void rowlse_accum(const DevStore& st, RowPart& p, int64_t row, bool row_ok,
                                             int64_t c0, int64_t ncols, const float* x) {
#pragma unroll
    for (int i = 0; i < W; ++i) {
        if (c0 + i < ncols) {
            const int q = __ldg(st.map + c0 + i);
            if (q != p.pid) {
                rowpart_flush(st, p, row, row_ok, true);
                p.pid = q;
                p.acc = 0.0f;
                p.mx = -INFINITY;
            }
            const float mn = fmaxf(p.mx, x[i]);
            const float sc = (p.mx == -INFINITY) ? 0.0f : __expf(p.mx - mn);
            p.acc = p.acc * sc + __expf(x[i] - mn);
            p.mx = mn;
        }
    }
}

// Column sums of a 128-row x 32-column chunk, segmented by the row-piece map.
// Every epilogue thread deposits its row; warp quadrant 0 walks the columns.
__device__ __forceinline__ void colsum_chunk(const DevStore& st, float* red, int lrow, int64_t m0, int M,
                                             int64_t gcol0, int N, const float* x, bool row_ok) {
#pragma unroll
    for (int i = 0; i < CHUNK; ++i) red[lrow * RED_LD + i] = row_ok ? x[i] : 0.0f;
    named_bar_sync(1, 32 * EPI_WARPS);
    if (lrow < 32) {
        const int c = lrow;
        const int64_t gc = gcol0 + c;
        if (gc < N) {
            const int rows = (int)((M - m0) < BM ? (M - m0) : BM);
            const int pfirst = __ldg(st.map + m0);
            const int plast = __ldg(st.map + m0 + rows - 1);
            float* out = static_cast<float*>(st.ptr);
            if (pfirst == plast) {
                float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
                int r = 0;
                for (; r + 4 <= rows; r += 4) {
                    s0 += red[(r + 0) * RED_LD + c];
                    s1 += red[(r + 1) * RED_LD + c];
                    s2 += red[(r + 2) * RED_LD + c];
                    s3 += red[(r + 3) * RED_LD + c];
                }
                for (; r < rows; ++r) s0 += red[r * RED_LD + c];
                out[(int64_t)pfirst * st.ld + gc] = (s0 + s1) + (s2 + s3);
            } else {
                int pid = pfirst;
                float s = 0.f;
                for (int r = 0; r < rows; ++r) {
                    const int q = __ldg(st.map + m0 + r);
                    if (q != pid) {
                        out[(int64_t)pid * st.ld + gc] = s;
                        pid = q;
                        s = 0.f;
                    }
                    s += red[r * RED_LD + c];
                }
                out[(int64_t)pid * st.ld + gc] = s;
            }
        }
    }
    named_bar_sync(1, 32 * EPI_WARPS);
}

// --------------------------------------------------------------- kernel
template <typename TS>
__global__ void __launch_bounds__(NUM_THREADS, 1)
coda_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                 const __grid_constant__ GemmParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
    float* red = reinterpret_cast<float*>(sB + STAGES * B_STAGE_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(red + BM * RED_LD);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 32 * EPI_WARPS);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tma_a);
        tma_prefetch_desc(&tma_b);
    }
    if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    griddep_launch_dependents();
    griddep_wait();

    const MainParams mp{P.M, P.N, P.K, P.ntm, P.ntn, P.nk, P.ntiles, P.a_mn, P.b_mn, 16,
                        P.ntiles, 0, 1, P.ntiles, 0, 0};
    auto tile_mn = [&](int t, int& tm, int& tn) { tile_coord(mp, t, tm, tn); };

    if (warp == 0) {
        producer_loop<1>(mp, &tma_a, &tma_b, sA, sB, full, empty, 0, blockIdx.x, gridDim.x);
    } else if (warp == 1) {
        mma_loop<1>(mp, tmem_base, sA, sB, full, empty, tfull, tempty, blockIdx.x, gridDim.x);
    } else {
        // ------------------------------------------------ epilogue
        const int q = warp & 3;                 // TMEM lane quadrant this warp may read
        const int lrow = q * 32 + lane;         // tile row owned by this thread
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < P.ntiles; t += gridDim.x) {
            int tm, tn;
            tile_mn(t, tm, tn);
            const int64_t m0 = (int64_t)tm * BM, n0 = (int64_t)tn * BN;
            const int64_t row = m0 + lrow;
            const bool row_ok = row < P.M;
            const int64_t rem_chunks = ((int64_t)P.N - n0 + CHUNK - 1) / CHUNK;
            const int nchunks = rem_chunks < BN / CHUNK ? (int)rem_chunks : BN / CHUNK;
            RowPart rp[MAX_ROW_STREAMS];
#pragma unroll
            for (int i = 0; i < MAX_ROW_STREAMS; ++i) rp[i] = RowPart{0.f, -INFINITY, -1};

            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);

            for (int j = 0; j < nchunks; ++j) {
                float v[64];
                {
                    float c[32];
                    tmem_ld32(tbase + j * CHUNK, c);
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = c[i];
                }
                if (j == nchunks - 1) {
                    // accumulator fully drained: hand the TMEM buffer back to the MMA warp
                    tc_fence_before();
                    mbar_arrive(&tempty[acc]);
                }
                const int64_t gcol0 = n0 + (int64_t)j * CHUNK;
                int w = CHUNK;
                if (P.acc_in != nullptr && row_ok) {
                    float x[32];
                    load_seg<float, 32>(P.acc_in + row * P.ld_acc, gcol0, P.N, x);
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] += x[i];
                }
                for (int s = 0; s < P.nsteps; ++s) {
                    const DevStep& st = P.steps[s];
                    switch (st.op) {
                    case OP_ROW_VEC_MUL: {
                        const DevOperand& o = P.opnd[st.a[0]];
                        const float* vp = static_cast<const float*>(o.ptr);
                        with_width(w, [&](auto wc) {
                            constexpr int W = decltype(wc)::value;
                            float g[W];
                            load_vec_seg<W>(vp, gcol0 * W / CHUNK, o.cols, g);
#pragma unroll
                            for (int i = 0; i < W; ++i) v[i] *= g[i];
                        });
                        break;
                    }
                    case OP_ROW_SCALE: {
                        const float* vp = static_cast<const float*>(P.opnd[st.a[0]].ptr);
                        float r = 0.0f;
                        if (row_ok) {
                            if (st.fin_src) {
                                const DevOperand& fp = P.opnd[st.fin_src - 1];
                                r = finalize_row(static_cast<const float*>(fp.ptr) + row * fp.ld, (int)fp.cols,
                                                 st.fin_kind, (float)st.fin_d, st.fin_eps);
                                if (n0 == 0 && j == 0) const_cast<float*>(vp)[row] = r;
                            } else {
                                r = __ldg(vp + row);
                            }
                        }
#pragma unroll
                        for (int i = 0; i < 64; ++i) v[i] *= r;
                        break;
                    }
                    case OP_RESIDUAL_ADD: {
                        const DevOperand& o = P.opnd[st.a[0]];
                        if (row_ok) {
                            const TS* rp_ = static_cast<const TS*>(o.ptr) + row * o.ld;
                            with_width(w, [&](auto wc) {
                                constexpr int W = decltype(wc)::value;
                                float x[W];
                                load_seg<TS, W>(rp_, gcol0 * W / CHUNK, o.cols, x);
#pragma unroll
                                for (int i = 0; i < W; ++i) v[i] += x[i];
                            });
                        }
                        break;
                    }
                    case OP_AUX_TILE_STORE: {
                        const DevStore& o = P.store[st.a[0]];
                        if (row_ok) {
                            TS* rp_ = static_cast<TS*>(o.ptr) + row * o.ld;
                            with_width(w, [&](auto wc) {
                                constexpr int W = decltype(wc)::value;
                                store_seg<TS, W>(rp_, gcol0 * W / CHUNK, o.cols, v);
                            });
                        }
                        break;
                    }
                    case OP_PARTIAL_SUMSQ: {
                        float x[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) x[i] = v[i] * v[i];
                        const DevStore& o = P.store[st.a[0]];
                        rowsum_accum<32>(o, rp[st.a[6]], row, row_ok, gcol0, P.N, x);
                        break;
                    }
                    case OP_PARTIAL_ROWDOT: {
                        const DevOperand& oi = P.opnd[st.a[0]];
                        float x[32];
                        if (row_ok) load_seg<TS, 32>(static_cast<const TS*>(oi.ptr) + row * oi.ld, gcol0, oi.cols, x);
                        else {
#pragma unroll
                            for (int i = 0; i < 32; ++i) x[i] = 0.f;
                        }
#pragma unroll
                        for (int i = 0; i < 32; ++i) x[i] *= v[i];
                        const DevStore& o = P.store[st.a[1]];
                        rowsum_accum<32>(o, rp[st.a[6]], row, row_ok, gcol0, P.N, x);
                        break;
                    }
                    case OP_PARTIAL_COLSUM: {
                        colsum_chunk(P.store[st.a[0]], red, lrow, m0, P.M, gcol0, P.N, v, row_ok);
                        break;
                    }
                    case OP_ONLINE_LSE: {
                        const DevStore& o = P.store[st.a[0]];
                        rowlse_accum<32>(o, rp[st.a[6]], row, row_ok, gcol0, P.N, v);
                        break;
                    }
                    case OP_TARGET_GATHER: {
                        if (row_ok) {
                            const int64_t lab = static_cast<const int64_t*>(P.opnd[st.a[0]].ptr)[row];
                            const int64_t local = lab - gcol0;
                            if (local >= 0 && local < 32 && lab < P.N) {
                                float val = 0.f;
#pragma unroll
                                for (int i = 0; i < 32; ++i)
                                    if (i == (int)local) val = v[i];
                                static_cast<float*>(P.store[st.a[1]].ptr)[row] = val;
                            }
                        }
                        break;
                    }
                    case OP_ROPE: {
                        const DevOperand& oc = P.opnd[st.a[0]];
                        const DevOperand& os = P.opnd[st.a[1]];
                        const float sgn = st.a[2] ? -1.0f : 1.0f;
                        if (row_ok) {
                            const TS* cp = static_cast<const TS*>(oc.ptr) + row * oc.ld;
                            const TS* sp = static_cast<const TS*>(os.ptr) + row * os.ld;
                            with_width(w, [&](auto wc) {
                                constexpr int W = decltype(wc)::value;
                                if constexpr (W >= 2) {
                                    float cs[W], sn[W];
                                    load_seg<TS, W>(cp, gcol0 * W / CHUNK, oc.cols, cs);
                                    load_seg<TS, W>(sp, gcol0 * W / CHUNK, os.cols, sn);
#pragma unroll
                                    for (int k = 0; k < W / 2; ++k) {
                                        const float x0 = v[2 * k], x1 = v[2 * k + 1];
                                        const float se = sgn * sn[2 * k], so = sgn * sn[2 * k + 1];
                                        v[2 * k] = x0 * cs[2 * k] - x1 * se;
                                        v[2 * k + 1] = x0 * so + x1 * cs[2 * k + 1];
                                    }
                                }
                            });
                        }
                        break;
                    }
                    case OP_SWIGLU: {
                        // pairs (2k, 2k+1) -> k; w >= 2 (validated on the host)
#pragma unroll
                        for (int k = 0; k < 32; ++k) {
                            if (2 * k < w) {
                                const float g = v[2 * k], u = v[2 * k + 1];
                                v[k] = g * sigmoid_stable(g) * u;
                            }
                        }
                        w >>= 1;
                        break;
                    }
                    case OP_SWIGLU_BWD: {
                        // entry width 32 (factor 1); preact read at 64 (factor 2)
                        const DevOperand& oz = P.opnd[st.a[0]];
                        float z[64];
                        if (row_ok) load_seg<TS, 64>(static_cast<const TS*>(oz.ptr) + row * oz.ld, gcol0 * 2, oz.cols, z);
                        else {
#pragma unroll
                            for (int i = 0; i < 64; ++i) z[i] = 0.f;
                        }
                        float rec[32];
                        // descending k: v[2k], v[2k+1] overwrite only entries >= k
#pragma unroll
                        for (int k = 31; k >= 0; --k) {
                            const float g = z[2 * k], u = z[2 * k + 1], d = v[k];
                            const float sg = sigmoid_stable(g);
                            const float sl = g * sg;
                            rec[k] = sl * u;
                            const float gu = d * sl;
                            const float gg = d * u * (sg + sl * (1.0f - sg));
                            v[2 * k] = gg;
                            v[2 * k + 1] = gu;
                            z[2 * k] = g * gg;        // <preact, grad_preact> terms
                            z[2 * k + 1] = u * gu;
                        }
                        const DevStore& orc = P.store[st.a[1]];
                        if (row_ok) store_seg<TS, 32>(static_cast<TS*>(orc.ptr) + row * orc.ld, gcol0, orc.cols, rec);
                        const DevStore& opd = P.store[st.a[2]];
                        rowsum_accum<64>(opd, rp[st.a[6]], row, row_ok, gcol0 * 2, (int64_t)P.N * 2, z);
                        w = 64;
                        break;
                    }
                    case OP_RMSNORM_BWD: {
                        const DevOperand& op_pre = P.opnd[st.a[0]];
                        float cpre[32], gam[32];
                        float r = 0.f, sstat = 0.f;
                        if (row_ok) {
                            load_seg<TS, 32>(static_cast<const TS*>(op_pre.ptr) + row * op_pre.ld, gcol0, op_pre.cols, cpre);
                            r = __ldg(static_cast<const float*>(P.opnd[st.a[1]].ptr) + row);
                            float* sp_ = static_cast<float*>(const_cast<void*>(P.opnd[st.a[3]].ptr));
                            if (st.fin_src) {
                                const DevOperand& fp = P.opnd[st.fin_src - 1];
                                sstat = finalize_row(static_cast<const float*>(fp.ptr) + row * fp.ld, (int)fp.cols,
                                                     st.fin_kind, (float)st.fin_d, st.fin_eps);
                                if (n0 == 0 && j == 0) sp_[row] = sstat;
                            } else {
                                sstat = __ldg(sp_ + row);
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < 32; ++i) cpre[i] = 0.f;
                        }
                        load_vec_seg<32>(static_cast<const float*>(P.opnd[st.a[2]].ptr), gcol0, P.opnd[st.a[2]].cols, gam);
                        float tmp[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            cpre[i] *= r;                 // c_n = c * r
                            tmp[i] = cpre[i] * gam[i];    // normed = c_n * gamma
                        }
                        const DevStore& on = P.store[st.a[5]];
                        if (row_ok) store_seg<TS, 32>(static_cast<TS*>(on.ptr) + row * on.ld, gcol0, on.cols, tmp);
#pragma unroll
                        for (int i = 0; i < 32; ++i) tmp[i] = v[i] * cpre[i];   // D * c_n
                        colsum_chunk(P.store[st.a[6]], red, lrow, m0, P.M, gcol0, P.N, tmp, row_ok);
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = (v[i] * gam[i] - cpre[i] * sstat) * r;
                        if (st.a[4] >= 0 && row_ok) {
                            const DevOperand& oa = P.opnd[st.a[4]];
                            float x[32];
                            load_seg<TS, 32>(static_cast<const TS*>(oa.ptr) + row * oa.ld, gcol0, oa.cols, x);
#pragma unroll
                            for (int i = 0; i < 32; ++i) v[i] += x[i];
                        }
                        break;
                    }
                    case OP_XENT_BWD: {
                        // d loss / d logits = (exp(x - lse) - onehot(label)) * scale; partials of x * grad
                        float lse_r = 0.0f;
                        int64_t lab = -1;
                        if (row_ok) {
                            lse_r = __ldg(static_cast<const float*>(P.opnd[st.a[0]].ptr) + row);
                            lab = static_cast<const int64_t*>(P.opnd[st.a[1]].ptr)[row];
                        }
                        const float gsc = __int_as_float(st.a[3]);
                        float x[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            float pr = __expf(v[i] - lse_r);
                            if (gcol0 + i == lab) pr -= 1.0f;
                            pr *= gsc;
                            x[i] = v[i] * pr;
                            v[i] = pr;
                        }
                        rowsum_accum<32>(P.store[st.a[2]], rp[st.a[6]], row, row_ok, gcol0, P.N, x);
                        break;
                    }
                    default:
                        break;
                    }
                }
                if (P.store_main && row_ok) {
                    const int64_t ncols = (int64_t)P.N * w / CHUNK;
                    with_width(w, [&](auto wc) {
                        constexpr int W = decltype(wc)::value;
                        const int64_t c0 = gcol0 * W / CHUNK;
                        if (P.out_f32)
                            store_seg<float, W>(static_cast<float*>(P.out) + row * P.ld_out, c0, ncols, v);
                        else
                            store_seg<__nv_bfloat16, W>(static_cast<__nv_bfloat16*>(P.out) + row * P.ld_out, c0,
                                                        ncols, v);
                    });
                }
            }
            // flush the row-directed partials of this tile (pieces end at tile edges)
            for (int s = 0; s < P.nsteps; ++s) {
                const DevStep& st = P.steps[s];
                int si = -1, slot = -1;
                bool pair = false;
                if (st.op == OP_PARTIAL_SUMSQ) { si = st.a[6]; slot = st.a[0]; }
                else if (st.op == OP_PARTIAL_ROWDOT) { si = st.a[6]; slot = st.a[1]; }
                else if (st.op == OP_ONLINE_LSE) { si = st.a[6]; slot = st.a[0]; pair = true; }
                else if (st.op == OP_SWIGLU_BWD) { si = st.a[6]; slot = st.a[2]; }
                else if (st.op == OP_XENT_BWD) { si = st.a[6]; slot = st.a[2]; }
                if (si >= 0 && si < MAX_ROW_STREAMS) rowpart_flush(P.store[slot], rp[si], row, row_ok, pair);
            }
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    }

    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}

constexpr size_t gemm_smem_bytes() {
    return 1024 + (size_t)STAGES * STAGE_BYTES + (size_t)BM * RED_LD * 4 + (2 * STAGES + 4) * 8 + 16;
}

}  // namespace coda
