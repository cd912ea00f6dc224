// coda_aux.cuh — the HBM-bound kernels around the fused GEMMs:
//   second-level reductions (reductions.py:64-168), the boundary RoPE
//   backward pass (kernels.py:560-617), piece->block folds, the SIM32
//   operand split and f32->bf16 storage conversion.
// All reductions run in a fixed ascending order with no atomics, so every
// launch is bit-reproducible (reductions.py:1-12).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include "coda_gemm.cuh"
#include "coda_ptx.cuh"

namespace coda {

// Row totals of (m, nb) partials in ascending block order.  A CTA stages 32
// rows through shared memory with coalesced loads, then thread r sums row r
// sequentially — the float32 op order of reductions.py:_row_sum_total.
constexpr int FIN_ROWS = 32;
constexpr int FIN_MAXNB = 512;

__device__ __forceinline__ float staged_row_total(const float* __restrict__ p, int64_t m, int64_t nb, int64_t ld,
                                                  float* tile, int64_t row0) {
    for (int64_t idx = threadIdx.x; idx < (int64_t)FIN_ROWS * nb; idx += blockDim.x) {
        const int64_t r = idx / nb, b = idx % nb;
        tile[r * (nb + 1) + b] = (row0 + r < m) ? p[(row0 + r) * ld + b] : 0.0f;
    }
    __syncthreads();
    float t = 0.0f;
    if (threadIdx.x < FIN_ROWS) {
        const float* row = tile + threadIdx.x * (nb + 1);
        for (int64_t b = 0; b < nb; ++b) t = __fadd_rn(t, row[b]);
    }
    return t;
}

// r = 1 / sqrt(total / d + eps) with IEEE-rounded intrinsics (reductions.py:74-78).
__global__ void coda_finalize_rms_kernel(const float* __restrict__ p, int64_t m, int64_t nb, int64_t ld,
                                         float d, float eps, float* __restrict__ r) {
    extern __shared__ float tile[];
    griddep_wait();
    griddep_launch_dependents();
    const int64_t row0 = (int64_t)blockIdx.x * FIN_ROWS;
    const float t = staged_row_total(p, m, nb, ld, tile, row0);
    if (threadIdx.x < FIN_ROWS && row0 + threadIdx.x < m)
        r[row0 + threadIdx.x] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(t, d), eps)));
}

__global__ void coda_finalize_rowdot_kernel(const float* __restrict__ p, int64_t m, int64_t nb, int64_t ld,
                                            float d, float* __restrict__ s) {
    extern __shared__ float tile[];
    griddep_wait();
    griddep_launch_dependents();
    const int64_t row0 = (int64_t)blockIdx.x * FIN_ROWS;
    const float t = staged_row_total(p, m, nb, ld, tile, row0);
    if (threadIdx.x < FIN_ROWS && row0 + threadIdx.x < m) s[row0 + threadIdx.x] = __fdiv_rn(t, d);
}

// Very wide partial rows (tiny reduction blocks): one thread per row, same order.
__global__ void coda_finalize_rms_wide_kernel(const float* __restrict__ p, int64_t m, int64_t nb, int64_t ld, float d,
                                              float eps, float* __restrict__ r) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    float t = 0.0f;
    for (int64_t b = 0; b < nb; ++b) t = __fadd_rn(t, p[i * ld + b]);
    r[i] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(t, d), eps)));
}

__global__ void coda_finalize_rowdot_wide_kernel(const float* __restrict__ p, int64_t m, int64_t nb, int64_t ld,
                                                 float d, float* __restrict__ s) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    float t = 0.0f;
    for (int64_t b = 0; b < nb; ++b) t = __fadd_rn(t, p[i * ld + b]);
    s[i] = __fdiv_rn(t, d);
}

// Column totals over tile rows (coalesced: one thread per column), summed in ascending
// row order; 16 rows of loads are issued ahead of each run of sequential adds.
__global__ void __launch_bounds__(64) coda_reduce_row_partials_kernel(const float* __restrict__ p, int64_t tm,
                                                                      int64_t n, int64_t ld, float* __restrict__ out) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    float t = 0.0f;
    int64_t b = 0;
    for (; b + 16 <= tm; b += 16) {
        float x[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = __ldg(p + (b + k) * ld + j);
#pragma unroll
        for (int k = 0; k < 16; ++k) t = __fadd_rn(t, x[k]);
    }
    for (; b < tm; ++b) t = __fadd_rn(t, p[b * ld + j]);
    out[j] = t;
}

__device__ __forceinline__ void lse_merge(float& m, float& s, float mb, float sb) {
    const float mn = fmaxf(m, mb);
    const float so = (m == -INFINITY) ? 0.0f : expf(m - mn);
    const float sn = (mb == -INFINITY) ? 0.0f : expf(mb - mn);
    s = s * so + sb * sn;
    m = mn;
}

// One thread per row, blocks merged strictly in ascending order (reductions.py:101-131).
// The merge chain is sequential, so the loads run ahead of it: 8 (max, sum) pairs per
// chunk as four 16-B loads, the next chunk in flight while the current one is merged
// (one row at a time and one pair per iteration, the round-1 loop waited on every load:
// 74 us for the LM head's 16384 x 256 pairs, 33.5 MB).
__global__ void __launch_bounds__(64) coda_combine_lse_kernel(const float* __restrict__ p, int64_t m, int64_t nb,
                                                              int64_t ld, float* __restrict__ lse) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const float* row = p + i * ld;
    float mx = -INFINITY, s = 0.0f;
    int64_t b = 0;
    if ((reinterpret_cast<uintptr_t>(row) & 15) == 0) {
        const float4* v = reinterpret_cast<const float4*>(row);
        const int64_t nc = nb / 8;   // whole chunks of 8 pairs
        float4 cur[4], nxt[4];
        if (nc > 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) cur[k] = __ldg(v + k);
        }
        for (int64_t c = 0; c < nc; ++c) {
            if (c + 1 < nc) {
#pragma unroll
                for (int k = 0; k < 4; ++k) nxt[k] = __ldg(v + 4 * (c + 1) + k);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                lse_merge(mx, s, cur[k].x, cur[k].y);
                lse_merge(mx, s, cur[k].z, cur[k].w);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) cur[k] = nxt[k];
        }
        b = nc * 8;
    }
    for (; b < nb; ++b) lse_merge(mx, s, row[2 * b], row[2 * b + 1]);
    lse[i] = (mx == -INFINITY) ? NAN : mx + logf(s);
}

__global__ void coda_ce_finalize_kernel(const float* __restrict__ target, const float* __restrict__ lse, int64_t m,
                                   float* __restrict__ loss) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) loss[i] = lse[i] - target[i];
}

// pieces (m, np) -> blocks (m, nb): block b sums pieces [ptr[b], ptr[b+1]).
__global__ void coda_combine_row_pieces_kernel(const float* __restrict__ pc, int64_t m, int64_t np, int64_t ldp,
                                          const int32_t* __restrict__ ptr, int64_t nb, int pairs,
                                          float* __restrict__ out, int64_t ldo) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= m * nb) return;
    const int64_t i = idx / nb, b = idx % nb;
    const float* row = pc + i * ldp;
    if (!pairs) {
        float t = 0.0f;
        for (int p = ptr[b]; p < ptr[b + 1]; ++p) t += row[p];
        out[i * ldo + b] = t;
    } else {
        float mx = -INFINITY, s = 0.0f;
        for (int p = ptr[b]; p < ptr[b + 1]; ++p) lse_merge(mx, s, row[2 * p], row[2 * p + 1]);
        out[i * ldo + 2 * b] = mx;
        out[i * ldo + 2 * b + 1] = s;
    }
}

// pieces (np, n) -> blocks (nb, n)
__global__ void coda_combine_col_pieces_kernel(const float* __restrict__ pc, int64_t np, int64_t n, int64_t ldp,
                                          const int32_t* __restrict__ ptr, int64_t nb,
                                          float* __restrict__ out, int64_t ldo) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    if (j >= n || b >= nb) return;
    float t = 0.0f;
    for (int p = ptr[b]; p < ptr[b + 1]; ++p) t += pc[(int64_t)p * ldp + j];
    out[b * ldo + j] = t;
}

// Boundary RoPE backward (kernels.py:589-606).  One CTA per row:
//   grad_z[2k]   =  g0*cos[2k]   + g1*sin[2k]
//   grad_z[2k+1] = -g0*sin[2k+1] + g1*cos[2k+1]
//   rowdot[b]    = sum_{c in block b} grad[c] * rotated[c]   (ascending c)
// The products are staged in shared memory so each block is reduced by one
// thread in column order (deterministic, no atomics).
template <typename TS>
__global__ void __launch_bounds__(256)
coda_rope_backward_stat_kernel(const TS* __restrict__ g, int64_t ldg, const TS* __restrict__ rot, int64_t ldr,
                          const TS* __restrict__ cs, int64_t ldc, const TS* __restrict__ sn, int64_t lds,
                          int64_t n, const int32_t* __restrict__ bstart, int64_t nb,
                          TS* __restrict__ gz, int64_t ldz, float* __restrict__ rowdot, int64_t ldd) {
    griddep_wait();
    griddep_launch_dependents();
    extern __shared__ float prod[];
    const int64_t i = blockIdx.x;
    constexpr int V = Io<TS>::V;
    const TS* gr = g + i * ldg;
    const TS* rr = rot + i * ldr;
    const TS* cr = cs + i * ldc;
    const TS* sr = sn + i * lds;
    TS* zr = gz + i * ldz;
    for (int64_t c0 = (int64_t)threadIdx.x * V; c0 < n; c0 += (int64_t)blockDim.x * V) {
        float gv[V], rv[V], cv[V], sv[V], zv[V];
        if (c0 + V <= n) {
            Io<TS>::load(gr + c0, gv);
            Io<TS>::load(rr + c0, rv);
            Io<TS>::load(cr + c0, cv);
            Io<TS>::load(sr + c0, sv);
        } else {
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const bool ok = c0 + e < n;
                gv[e] = ok ? Io<TS>::load1(gr + c0 + e) : 0.f;
                rv[e] = ok ? Io<TS>::load1(rr + c0 + e) : 0.f;
                cv[e] = ok ? Io<TS>::load1(cr + c0 + e) : 0.f;
                sv[e] = ok ? Io<TS>::load1(sr + c0 + e) : 0.f;
            }
        }
#pragma unroll
        for (int k = 0; k < V / 2; ++k) {
            const float g0 = gv[2 * k], g1 = gv[2 * k + 1];
            zv[2 * k] = g0 * cv[2 * k] + g1 * sv[2 * k];
            zv[2 * k + 1] = -g0 * sv[2 * k + 1] + g1 * cv[2 * k + 1];
        }
#pragma unroll
        for (int e = 0; e < V; ++e)
            if (c0 + e < n) prod[c0 + e] = gv[e] * rv[e];
        store_seg<TS, V>(zr, c0, n, zv);
    }
    __syncthreads();
    for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) {
        float t = 0.0f;
        for (int c = bstart[b]; c < bstart[b + 1]; ++c) t += prod[c];
        rowdot[i * ldd + b] = t;
    }
}

// Fast path of the boundary RoPE backward for the default reduction layout
// (blocks of exactly 128 columns, the last one possibly ragged): no shared
// memory, every thread owns one 16-byte vector per 2048-column sweep, and the
// 128/V lanes covering one block reduce their partial dots with a shuffle
// tree.  Several rows per CTA keep enough loads in flight for HBM.
template <typename TS>
__global__ void __launch_bounds__(256)
coda_rope_backward_stat128_kernel(const TS* __restrict__ g, int64_t ldg, const TS* __restrict__ rot, int64_t ldr,
                             const TS* __restrict__ cs, int64_t ldc, const TS* __restrict__ sn, int64_t lds,
                             int64_t m, int64_t n, TS* __restrict__ gz, int64_t ldz, float* __restrict__ rowdot,
                             int64_t ldd) {
    griddep_wait();
    griddep_launch_dependents();
    constexpr int V = Io<TS>::V;
    constexpr int LPB = 128 / V;                       // lanes per 128-column block
    const int lane = threadIdx.x & 31;
    const int64_t sweep = (int64_t)blockDim.x * V;
    for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
        const TS* gr = g + i * ldg;
        const TS* rr = rot + i * ldr;
        const TS* cr = cs + i * ldc;
        const TS* sr = sn + i * lds;
        TS* zr = gz + i * ldz;
        for (int64_t base = 0; base < n; base += sweep) {
            const int64_t c0 = base + (int64_t)threadIdx.x * V;
            const bool ok = c0 < n;
            float gv[V], rv[V], cv[V], sv[V], zv[V];
            float p = 0.0f;
            if (ok) {
                if (c0 + V <= n) {
                    Io<TS>::load(gr + c0, gv);
                    Io<TS>::load(rr + c0, rv);
                    Io<TS>::load(cr + c0, cv);
                    Io<TS>::load(sr + c0, sv);
                } else {
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        const bool in = c0 + e < n;
                        gv[e] = in ? Io<TS>::load1(gr + c0 + e) : 0.f;
                        rv[e] = in ? Io<TS>::load1(rr + c0 + e) : 0.f;
                        cv[e] = in ? Io<TS>::load1(cr + c0 + e) : 0.f;
                        sv[e] = in ? Io<TS>::load1(sr + c0 + e) : 0.f;
                    }
                }
#pragma unroll
                for (int k = 0; k < V / 2; ++k) {
                    const float g0 = gv[2 * k], g1 = gv[2 * k + 1];
                    zv[2 * k] = g0 * cv[2 * k] + g1 * sv[2 * k];
                    zv[2 * k + 1] = -g0 * sv[2 * k + 1] + g1 * cv[2 * k + 1];
                }
#pragma unroll
                for (int e = 0; e < V; ++e) p += gv[e] * rv[e];
                store_seg<TS, V>(zr, c0, n, zv);
            }
#pragma unroll
            for (int off = LPB / 2; off >= 1; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
            if (ok && (lane % LPB) == 0) rowdot[i * ldd + c0 / 128] = p;
        }
    }
}

// Compact-table variant (bf16): cs/sn are (m, h/2) with one angle per pair; columns
// [0, 2h) rotate by pair (col mod h)/2 (q and k spans share angles), columns >= 2h are the
// identity.  Reads 2 x m x h bytes of tables instead of 4 x m x n; arithmetic identical.
__global__ void __launch_bounds__(256)
coda_rope_backward_stat128_compact_kernel(const __nv_bfloat16* __restrict__ g, int64_t ldg,
                                          const __nv_bfloat16* __restrict__ rot, int64_t ldr,
                                          const __nv_bfloat16* __restrict__ cs, int64_t ldc,
                                          const __nv_bfloat16* __restrict__ sn, int64_t lds, int64_t h,
                                          int64_t m, int64_t n, __nv_bfloat16* __restrict__ gz, int64_t ldz,
                                          float* __restrict__ rowdot, int64_t ldd) {
    griddep_wait();
    griddep_launch_dependents();
    using TS = __nv_bfloat16;
    constexpr int V = Io<TS>::V;                       // 8
    constexpr int LPB = 128 / V;
    constexpr int U = 1;                               // sweeps per iteration (2 measured slower: registers)
    const int lane = threadIdx.x & 31;
    const int64_t sweep = (int64_t)blockDim.x * V;
    for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
        const TS* gr = g + i * ldg;
        const TS* rr = rot + i * ldr;
        const TS* cr = cs + i * ldc;
        const TS* sr = sn + i * lds;
        TS* zr = gz + i * ldz;
        for (int64_t base = 0; base < n; base += U * sweep) {
            float gv[U][V], rv[U][V], cv[U][V], sv[U][V];
            int64_t c0[U];
            bool ok[U];
            // issue every load of U sweeps before any arithmetic
#pragma unroll
            for (int u = 0; u < U; ++u) {
                c0[u] = base + u * sweep + (int64_t)threadIdx.x * V;
                ok[u] = c0[u] < n;
                if (ok[u] && c0[u] + V <= n) {
                    Io<TS>::load(gr + c0[u], gv[u]);
                    Io<TS>::load(rr + c0[u], rv[u]);
                } else {
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        const bool in = ok[u] && c0[u] + e < n;
                        gv[u][e] = in ? Io<TS>::load1(gr + c0[u] + e) : 0.f;
                        rv[u][e] = in ? Io<TS>::load1(rr + c0[u] + e) : 0.f;
                    }
                }
                if (ok[u] && c0[u] < 2 * h) {
                    const int64_t p0 = (c0[u] % h) / 2;     // multiple of 4: h % 32 == 0, c0 % 8 == 0
                    const uint2 uc = __ldg(reinterpret_cast<const uint2*>(cr + p0));
                    const uint2 us = __ldg(reinterpret_cast<const uint2*>(sr + p0));
                    const uint32_t wc[2] = {uc.x, uc.y}, ws[2] = {us.x, us.y};
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const float c_lo = __uint_as_float(wc[j] << 16), c_hi = __uint_as_float(wc[j] & 0xFFFF0000u);
                        const float s_lo = __uint_as_float(ws[j] << 16), s_hi = __uint_as_float(ws[j] & 0xFFFF0000u);
                        cv[u][4 * j] = cv[u][4 * j + 1] = c_lo;
                        cv[u][4 * j + 2] = cv[u][4 * j + 3] = c_hi;
                        sv[u][4 * j] = sv[u][4 * j + 1] = s_lo;
                        sv[u][4 * j + 2] = sv[u][4 * j + 3] = s_hi;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        cv[u][e] = 1.0f;
                        sv[u][e] = 0.0f;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float zv[V];
                float p = 0.0f;
#pragma unroll
                for (int k = 0; k < V / 2; ++k) {
                    const float g0 = gv[u][2 * k], g1 = gv[u][2 * k + 1];
                    zv[2 * k] = g0 * cv[u][2 * k] + g1 * sv[u][2 * k];
                    zv[2 * k + 1] = -g0 * sv[u][2 * k + 1] + g1 * cv[u][2 * k + 1];
                }
#pragma unroll
                for (int e = 0; e < V; ++e) p += gv[u][e] * rv[u][e];
                if (ok[u]) store_seg<TS, V>(zr, c0[u], n, zv);
#pragma unroll
                for (int off = LPB / 2; off >= 1; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
                if (ok[u] && (lane % LPB) == 0) rowdot[i * ldd + c0[u] / 128] = p;
            }
        }
    }
}

// Compact-table boundary RoPE backward, deep-load variant (bf16, default 128-column blocks,
// n % (RBD_U * 2048) == 0, h % 32 == 0).  The plain compact kernel holds one 16-B vector of
// each operand per thread in flight and is latency-bound under the power cap (0.6 of HBM).
// Here every thread first issues RBD_U independent 16-B loads of grad and of rotated (kept as
// raw bf16 words, 8 registers each) plus their table words, then converts and computes, so
// ~3-6x the bytes are in flight per thread (RBD_U = 3 or 6 sweeps; streaming, L1-bypassing
// loads and stores).  Same arithmetic and
// reduction order as coda_rope_backward_stat128_compact_kernel.
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int RBD_U>
__global__ void __launch_bounds__(256)
coda_rope_backward_stat_deep_kernel(const __nv_bfloat16* __restrict__ g, int64_t ldg,
                                    const __nv_bfloat16* __restrict__ rot, int64_t ldr,
                                    const __nv_bfloat16* __restrict__ cs, int64_t ldc,
                                    const __nv_bfloat16* __restrict__ sn, int64_t lds, int64_t h,
                                    int64_t m, int64_t n, __nv_bfloat16* __restrict__ gz, int64_t ldz,
                                    float* __restrict__ rowdot, int64_t ldd) {
    griddep_wait();
    griddep_launch_dependents();
    using TS = __nv_bfloat16;
    const int lane = threadIdx.x & 31;
    constexpr int64_t SWEEP = 256 * 8;
    const int64_t per_row = n / (RBD_U * SWEEP);
    const int64_t total = m * per_row;
    for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
        const int64_t i = it / per_row;
        const int64_t base = (it - i * per_row) * (RBD_U * SWEEP);
        const TS* gr = g + i * ldg;
        const TS* rr = rot + i * ldr;
        uint4 gw[RBD_U], rw[RBD_U];
        uint2 cw[RBD_U], sw[RBD_U];
        int64_t c0[RBD_U];
#pragma unroll
        for (int u = 0; u < RBD_U; ++u) {
            c0[u] = base + u * SWEEP + (int64_t)threadIdx.x * 8;
            gw[u] = ld_stream_v4(gr + c0[u]);
            rw[u] = ld_stream_v4(rr + c0[u]);
            if (c0[u] < 2 * h) {
                const int64_t p0 = (c0[u] % h) / 2;
                cw[u] = __ldg(reinterpret_cast<const uint2*>(cs + i * ldc + p0));
                sw[u] = __ldg(reinterpret_cast<const uint2*>(sn + i * lds + p0));
            } else {
                cw[u] = make_uint2(0x3F803F80u, 0x3F803F80u);   // bf16 1.0 pairs
                sw[u] = make_uint2(0u, 0u);
            }
        }
#pragma unroll
        for (int u = 0; u < RBD_U; ++u) {
            const uint32_t gv_[4] = {gw[u].x, gw[u].y, gw[u].z, gw[u].w};
            const uint32_t rv_[4] = {rw[u].x, rw[u].y, rw[u].z, rw[u].w};
            const uint32_t wc[2] = {cw[u].x, cw[u].y}, ws[2] = {sw[u].x, sw[u].y};
            float gv[8], rv[8], cv[8], sv[8], zv[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                gv[2 * e] = __uint_as_float(gv_[e] << 16);
                gv[2 * e + 1] = __uint_as_float(gv_[e] & 0xFFFF0000u);
                rv[2 * e] = __uint_as_float(rv_[e] << 16);
                rv[2 * e + 1] = __uint_as_float(rv_[e] & 0xFFFF0000u);
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const float c_lo = __uint_as_float(wc[j] << 16), c_hi = __uint_as_float(wc[j] & 0xFFFF0000u);
                const float s_lo = __uint_as_float(ws[j] << 16), s_hi = __uint_as_float(ws[j] & 0xFFFF0000u);
                cv[4 * j] = cv[4 * j + 1] = c_lo;
                cv[4 * j + 2] = cv[4 * j + 3] = c_hi;
                sv[4 * j] = sv[4 * j + 1] = s_lo;
                sv[4 * j + 2] = sv[4 * j + 3] = s_hi;
            }
            float p = 0.0f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float g0 = gv[2 * k], g1 = gv[2 * k + 1];
                zv[2 * k] = g0 * cv[2 * k] + g1 * sv[2 * k];
                zv[2 * k + 1] = -g0 * sv[2 * k + 1] + g1 * cv[2 * k + 1];
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) p += gv[e] * rv[e];
            {
                uint4 o;
                o.x = pack_bf16x2(zv[0], zv[1]);
                o.y = pack_bf16x2(zv[2], zv[3]);
                o.z = pack_bf16x2(zv[4], zv[5]);
                o.w = pack_bf16x2(zv[6], zv[7]);
                __stcs(reinterpret_cast<uint4*>(gz + i * ldz + c0[u]), o);
            }
#pragma unroll
            for (int off = 8; off >= 1; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
            if ((lane & 15) == 0) rowdot[i * ldd + c0[u] / 128] = p;
        }
    }
}

// SIM32 split: x = x0 + x1 + x2 with x0 = bf16(x), x1 = bf16(x - x0), x2 = bf16(x - x0 - x1)
// (each difference is exact in f32).  dst holds 6 K-blocks of kp, block j = term pattern[j].
struct SplitPattern { int t[6]; };

__device__ __forceinline__ float split_term(float x, int term) {
    const float x0 = __bfloat162float(__float2bfloat16_rn(x));
    if (term == 0) return x0;
    const float r1 = x - x0;
    const float x1 = __bfloat162float(__float2bfloat16_rn(r1));
    if (term == 1) return x1;
    return r1 - x1;   // rounded to bf16 on store
}

__global__ void coda_split_operand_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                                     int k_axis, int64_t kp, SplitPattern pat,
                                     __nv_bfloat16* __restrict__ dst, int64_t drows, int64_t dcols, int64_t ldd) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= drows * dcols) return;
    const int64_t r = idx / dcols, c = idx % dcols;
    float val = 0.0f;
    if (k_axis == 1) {          // K along columns: dst (rows, 6kp)
        const int j = (int)(c / kp);
        const int64_t k = c % kp;
        if (k < cols) val = split_term(src[r * lds + k], pat.t[j]);
    } else {                    // K along rows: dst (6kp, cols)
        const int j = (int)(r / kp);
        const int64_t k = r % kp;
        if (k < rows) val = split_term(src[k * lds + c], pat.t[j]);
    }
    dst[r * ldd + c] = __float2bfloat16_rn(val);
}

__global__ void __launch_bounds__(256)
coda_convert_f32_bf16_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                             __nv_bfloat16* __restrict__ dst, int64_t ldd, int vec) {
    griddep_wait();
    griddep_launch_dependents();
    // 8 elements per thread step: two 16-B streaming loads, one 16-B store (when rows are
    // 16-B aligned: vec = 1); HBM-bound, 6 B per element.  Unaligned rows go scalar.
    const int64_t vpr = vec ? cols / 8 : 0;
    const int64_t total = rows * vpr;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += stride) {
        const int64_t r = v / vpr, c = (v - r * vpr) * 8;
        const float4 a = __ldcs(reinterpret_cast<const float4*>(src + r * lds + c));
        const float4 b = __ldcs(reinterpret_cast<const float4*>(src + r * lds + c + 4));
        uint4 o;
        o.x = pack_bf16x2(a.x, a.y);
        o.y = pack_bf16x2(a.z, a.w);
        o.z = pack_bf16x2(b.x, b.y);
        o.w = pack_bf16x2(b.z, b.w);
        __stcs(reinterpret_cast<uint4*>(dst + r * ldd + c), o);
    }
    const int64_t c0 = vpr * 8;
    if (c0 < cols) {
        for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride)
            for (int64_t c = c0; c < cols; ++c) dst[r * ldd + c] = __float2bfloat16_rn(src[r * lds + c]);
    }
}

// Row scaling of a bf16 matrix: dst[i, :] = bf16(scale[i] * src[i, :]) (RNE).  Folds an
// RMSNorm gain into the weight matrix that consumes the normalized rows,
// W' = diag(gamma) W, once per weight update.  HBM-bound: 4 B per element; 8 elements
// (one 16-B load and store) per thread step when rows are 16-B aligned.
__global__ void __launch_bounds__(256)
coda_scale_rows_kernel(const __nv_bfloat16* __restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                       const float* __restrict__ scale, __nv_bfloat16* __restrict__ dst, int64_t ldd, int vec) {
    griddep_wait();
    griddep_launch_dependents();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (vec) {
        const int64_t vpr = cols / 8;
        const int64_t total = rows * vpr;
        for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += stride) {
            const int64_t r = v / vpr, c = (v - r * vpr) * 8;
            const float g = __ldg(scale + r);
            float x[8];
            Io<__nv_bfloat16>::load(src + r * lds + c, x);
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] *= g;
            Io<__nv_bfloat16>::store(dst + r * ldd + c, x);
        }
        return;
    }
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < rows * cols; v += stride) {
        const int64_t r = v / cols, c = v - r * cols;
        dst[r * ldd + c] = __float2bfloat16_rn(__ldg(scale + r) * __bfloat162float(src[r * lds + c]));
    }
}

}  // namespace coda
