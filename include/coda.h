/*
 * coda.h — C-ABI of the B200-native CODA fused GEMM + epilogue engine.
 *
 * The reference (`tilefuse`, /root/reference/pkg/src/tilefuse) is a pure
 * Python/numpy package with no FFI.  Its drop-in boundary is the Python op /
 * epilogue-primitive API; the Python package `paper_2605_19269_b200` mirrors
 * that API and calls these entry points through ctypes.  Each entry point
 * below names the reference interface it replaces (file:line).
 *
 * Conventions
 *   - Plain pointers, sizes and strides; no torch types.  The caller owns and
 *     allocates every buffer (inputs, outputs, workspaces); the library never
 *     allocates device memory and only borrows pointers for the duration of the
 *     stream-ordered work it enqueues.
 *   - All work is asynchronous on the caller's `stream` (a cudaStream_t).
 *   - Return 0 on success, a negative CODA_E_* code on failure (validation
 *     happens before anything is enqueued).  coda_last_error() returns the
 *     thread-local message of the last failure.
 *   - 2-D tensors are row-major with leading dimension `ld` (elements); `ld`
 *     times the element size must be a multiple of 16 bytes and `ptr` must be
 *     16-byte aligned (TMA / vector-access requirement).
 */
#ifndef CODA_H
#define CODA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes: 1:1 with the reference taxonomy (errors.py:9-56) ---- */
#define CODA_OK                 0
#define CODA_E_DIMENSION       -1   /* DimensionError   errors.py:13 */
#define CODA_E_BINDING         -2   /* BindingError     errors.py:17 */
#define CODA_E_PROGRAM         -3   /* ProgramError     errors.py:21 */
#define CODA_E_PAIRING         -4   /* PairingError     errors.py:26 */
#define CODA_E_CONFIG          -5   /* ConfigError      errors.py:30 */
#define CODA_E_LABEL           -6   /* LabelError       errors.py:34 */
#define CODA_E_DEGENERATE      -7   /* DegenerateError  errors.py:42 */
#define CODA_E_CUDA            -20  /* device / launch failure */

/* ---- element types ---- */
#define CODA_BF16  0
#define CODA_F32   1
#define CODA_I64   2
#define CODA_I32   3

/* ---- epilogue op codes: one per reference primitive (epilogue.py:198-593) ---- */
#define CODA_OP_ROW_VEC_MUL      1   /* RowVecMul          epilogue.py:198 */
#define CODA_OP_ROW_SCALE        2   /* RowScale           epilogue.py:214 */
#define CODA_OP_RESIDUAL_ADD     3   /* ResidualAdd        epilogue.py:230 */
#define CODA_OP_AUX_TILE_STORE   4   /* AuxTileStore       epilogue.py:246 */
#define CODA_OP_PARTIAL_SUMSQ    5   /* PartialSumSq       epilogue.py:273 */
#define CODA_OP_PARTIAL_ROWDOT   6   /* PartialRowDot      epilogue.py:294 */
#define CODA_OP_PARTIAL_COLSUM   7   /* PartialColSum      epilogue.py:319 */
#define CODA_OP_ONLINE_LSE       8   /* OnlineLse          epilogue.py:338 */
#define CODA_OP_TARGET_GATHER    9   /* TargetGather       epilogue.py:373 */
#define CODA_OP_ROPE            10   /* PairwiseRope       epilogue.py:409 */
#define CODA_OP_SWIGLU          11   /* PairwiseSwiglu     epilogue.py:449 */
#define CODA_OP_SWIGLU_BWD      12   /* PairwiseSwigluBackward epilogue.py:469 */
#define CODA_OP_RMSNORM_BWD     13   /* RmsNormBackwardLocal   epilogue.py:522 */
#define CODA_OP_XENT_BWD        14   /* CrossEntropyBackward (B200 extension: softmax CE gradient) */

#define CODA_MAX_STEPS       16
#define CODA_MAX_OPERANDS    16
#define CODA_MAX_STORES      16
#define CODA_MAX_ROW_STREAMS  4
#define CODA_MAX_PEERS        8
#define CODA_FIN_RMS          1   /* coda_step_t.fin_kind: finalize_rms    reductions.py:64-80 */
#define CODA_FIN_ROWDOT       2   /*                       finalize_rowdot reductions.py:83-98 */   /* row-directed partial streams (sum / row-dot / LSE) per program */

/* A dense 1-D/2-D device tensor.  1-D tensors use rows = 1, cols = length. */
typedef struct {
    void*   ptr;
    int64_t rows;
    int64_t cols;
    int64_t ld;      /* leading dimension in elements (2-D) */
    int32_t dtype;   /* CODA_BF16 / CODA_F32 / CODA_I64 / CODA_I32 */
    int32_t _pad;
} coda_tensor_t;

/* One GEMM launch: GemmProblem (engine.py:55-76) after lowering.
 * storage: CODA_BF16 (SIMBF16) or CODA_F32 (SIM32; A/B are then the
 * 6-term bf16 split operands produced by coda_split_operand, k = 6*kp). */
typedef struct {
    int64_t m, n, k;
    int32_t trans_a, trans_b;
    int32_t storage;       /* dtype of side TILE operands and aux TILE stores */
    int32_t out_dtype;     /* dtype of the main output */
    int32_t store_main;    /* engine.py:428-430 */
    int32_t sm_limit;      /* 0: the persistent grid uses every SM; > 0: at most this many SMs,
                              leaving the rest to concurrent work on other streams (e.g. the
                              data-parallel weight-gradient all-reduce).  Results never change. */
    /* Optional caller-owned scratch for wave-tail splitting (split-K of the last,
     * partial wave).  Every K piece of a split tile dumps its f32 partial and arrives
     * on a counter; the last arrival sums all pieces in fixed piece order (bitwise
     * deterministic) and runs the program.  No piece waits for another, so nothing
     * assumes the launch's clusters are co-resident.  The first 64 KiB hold int32
     * counters that must be zero before the first launch (the kernels leave them
     * zero); the rest holds f32 partial tiles.  NULL / 0 disables splitting.
     * Launches sharing one workspace must be stream-ordered. */
    void*   workspace;
    int64_t workspace_bytes;
} coda_problem_t;

/* One program step (EpilogueProgram.steps, epilogue.py:606-698).
 * arg[] holds operand / store slot indices; meaning per op:
 *   ROW_VEC_MUL    arg0 = operand (row vector)
 *   ROW_SCALE      arg0 = operand (col vector)
 *   RESIDUAL_ADD   arg0 = operand (tile)
 *   AUX_TILE_STORE arg0 = store (tile)
 *   PARTIAL_SUMSQ  arg0 = store (row-sum pieces), arg6 = row stream
 *   PARTIAL_ROWDOT arg0 = operand (tile), arg1 = store (row-sum pieces), arg6 = row stream
 *   PARTIAL_COLSUM arg0 = store (col-sum pieces)
 *   ONLINE_LSE     arg0 = store (row-pair pieces), arg6 = row stream
 *   TARGET_GATHER  arg0 = operand (labels, int64), arg1 = store (gather, f32)
 *   ROPE           arg0 = cos operand, arg1 = sin operand, arg2 = backward flag,
 *                  arg3/arg4 = 1 + slot of compact (m, h/2) bf16 cos/sin tables or 0,
 *                  arg5 = h: column c < 2h rotates by angle (c mod h)/2, c >= 2h is the
 *                  identity; 2h <= n (packed qkv, q-span width h) or h == n (a plain table)
 *   SWIGLU         —
 *   SWIGLU_BWD     arg0 = preact operand (factor 2), arg1 = recompute store,
 *                  arg2 = row-sum pieces store (factor 2), arg6 = row stream
 *   RMSNORM_BWD    arg0 = pre, arg1 = inv_rms, arg2 = gamma, arg3 = stat,
 *                  arg4 = accumulate operand or -1, arg5 = normed store,
 *                  arg6 = gamma-grad col-sum pieces store
 *   XENT_BWD       arg0 = lse operand (col vector), arg1 = labels operand (int64),
 *                  arg2 = row-sum pieces store of sum(tile * grad), arg3 = grad_scale
 *                  (float bits), arg6 = row stream
 * Row streams (0 .. CODA_MAX_ROW_STREAMS-1) number the program's row-directed
 * partial emitters in order; each carries its own running block sum per row.
 * width: running width at step entry in values per 32 accumulator columns, i.e.
 * 32 x the reference's running width factor (epilogue.py:626-660): 64 (factor 2),
 * 32 (1), 16 (1/2) ... 1 (1/32).  Pairwise steps need width >= 2. */
typedef struct {
    int32_t op;
    int32_t width;
    int32_t arg[7];
    /* Deferred finalizer (B200 extension; values identical to the standalone launch):
     * fin_src = 1 + operand slot of an f32 (m, nb) partial-block matrix, or 0.  When set,
     * the step's column-vector operand (ROW_SCALE: arg0, RMSNORM_BWD: the stat, arg3) is
     * computed inside this launch from those partials -- fin_kind 1: finalize_rms
     * r = 1/sqrt(sum_b p / fin_d + fin_eps) (reductions.py:64-80), 2: finalize_rowdot
     * s = sum_b p / fin_d (reductions.py:83-98), same f32 op order -- and written back to
     * that operand's vector by the launch, so the separate finalize launch disappears. */
    int32_t fin_src;
    int32_t fin_kind;
    int32_t fin_d;
    float   fin_eps;
    int32_t _pad;
} coda_step_t;

/* A partial/aux output.  For row-sum / row-pair / col-sum stores the tensor is
 * the *piece* buffer and `piece_map` maps every scaled column (row-sum,
 * row-pair; length n*factor) or every row (col-sum; length m) to its piece
 * index.  Pieces are reference reduction blocks (epilogue.py:96-130) split at
 * GPU tile boundaries; coda_combine_* folds them into blocks when they differ. */
typedef struct {
    coda_tensor_t  t;
    const int32_t* piece_map;
    int32_t        kind;      /* 0 tile, 1 row-sum, 2 row-pair, 3 col-sum, 4 gather */
    int32_t        aligned;   /* row-sum/row-pair: every piece starts on a 32*factor column
                                 boundary; col-sum: every piece starts on a 32-row boundary.
                                 Enables the specialised epilogue kernels. */
} coda_store_t;

/* run_gemm (engine.py:376-464) / run_gemm_trans (engine.py:467-478):
 * one persistent tcgen05 GEMM whose epilogue executes `steps`. */
int coda_gemm_epilogue(const coda_problem_t* problem,
                       const coda_tensor_t* a, const coda_tensor_t* b,
                       const coda_step_t* steps, int nsteps,
                       const coda_tensor_t* operands, int noperands,
                       const coda_store_t* stores, int nstores,
                       const coda_tensor_t* main_out,      /* NULL iff !store_main */
                       const coda_tensor_t* acc_in,        /* NULL, or f32 (m, n) added to the
                                                              accumulator before step 0 (C += A*B) */
                       void* stream);

/* finalize_rms (reductions.py:64-80): r[i] = 1/sqrt(sum_b p[i,b] / d + eps). */
int coda_finalize_rms(const float* partials, int64_t m, int64_t nb, int64_t ld,
                      int64_t d, float eps, float* r, void* stream);

/* finalize_rowdot (reductions.py:83-98): s[i] = sum_b p[i,b] / d. */
int coda_finalize_rowdot(const float* partials, int64_t m, int64_t nb, int64_t ld,
                         int64_t d, float* s, void* stream);

/* reduce_row_partials (reductions.py:134-145): out[j] = sum_t p[t,j]. */
int coda_reduce_row_partials(const float* partials, int64_t tm, int64_t n, int64_t ld,
                             float* out, void* stream);

/* combine_lse (reductions.py:101-131): lse[i] from (max, sum) pairs. */
int coda_combine_lse(const float* pairs, int64_t m, int64_t nb, int64_t ld,
                     float* lse, void* stream);

/* cross_entropy_finalize (reductions.py:148-168): loss = lse - target. */
int coda_cross_entropy_finalize(const float* target, const float* lse, int64_t m,
                                float* losses, void* stream);

/* rope_backward_stat (kernels.py:560-617): counter-rotated gradient (storage
 * dtype) plus row-dot partials of grad*rotated over row_block_layout
 * (`block_start`, nb+1 device offsets: block b covers [start[b], start[b+1])).
 * block_start == NULL selects the uniform 128-column layout (the default
 * tile_n = reduction_tile_n = 128), served by a shared-memory-free kernel. */
int coda_rope_backward_stat(const coda_tensor_t* grad, const coda_tensor_t* rotated,
                            const coda_tensor_t* cos, const coda_tensor_t* sin,
                            const int32_t* block_start, int64_t nb,
                            coda_tensor_t* grad_z, float* rowdot, int64_t ld_rowdot,
                            void* stream);

/* rope_backward_stat with compact tables (bf16, default 128-column row blocks):
 * cos_c / sin_c are (m, h/2), one angle per pair; grad columns [0, 2h) rotate by
 * pair (col mod h)/2 (the q and k spans of the packed projection share angles,
 * kernels.py:184-206) and columns >= 2h are the identity (the v span).  Same
 * results as coda_rope_backward_stat on the expanded (m, n) tables, with 2*m*h
 * instead of 4*m*n bytes of table reads.  h % 32 == 0, 2h <= n. */
int coda_rope_backward_stat_compact(const coda_tensor_t* grad, const coda_tensor_t* rotated,
                                    const coda_tensor_t* cos_c, const coda_tensor_t* sin_c, int64_t h,
                                    coda_tensor_t* grad_z, float* rowdot, int64_t ld_rowdot, void* stream);

/* Fold piece partials into reference blocks in ascending piece order.
 * block_ptr (nb+1, host-built CSR) lists the piece range of each block. */
int coda_combine_row_pieces(const float* pieces, int64_t m, int64_t np, int64_t ld_p,
                            const int32_t* block_ptr, int64_t nb, int pairs,
                            float* out, int64_t ld_o, void* stream);
int coda_combine_col_pieces(const float* pieces, int64_t np, int64_t n, int64_t ld_p,
                            const int32_t* block_ptr, int64_t nb,
                            float* out, int64_t ld_o, void* stream);

/* SIM32 operand preparation: splits an f32 operand into three bf16 terms
 * x = x0 + x1 + x2 and lays out six K-blocks so that one bf16 GEMM with
 * k' = 6*kp reproduces the f32 product to ~2^-24 (terms with i+j <= 2).
 * k_axis: 1 if K runs along columns (A, or trans_b B), 0 if along rows.
 * pattern: term index for each of the 6 K-blocks. */
int coda_split_operand(const coda_tensor_t* src, int k_axis, int64_t kp,
                       const int32_t pattern[6], coda_tensor_t* dst, void* stream);

/* Elementwise storage conversion f32 -> bf16 (RNE), used after an f32
 * allreduce of weight gradients so rounding happens once (engine.py:443-447). */
int coda_convert_f32_bf16(const coda_tensor_t* src, coda_tensor_t* dst, void* stream);

/* Gain folding (north_star "gamma folded into W"; B200 extension, no reference
 * counterpart): dst[i, :] = bf16(scale[i] * src[i, :]), bf16 (rows, cols) src/dst,
 * f32 scale[rows].  W' = diag(gamma) W is formed once per weight update, so the
 * producing launch (gemm_residual_partial_rms, kernels.py:325-360) no longer
 * multiplies by gamma nor stores the gained copy of its output. */
int coda_scale_rows(const coda_tensor_t* src, const float* scale, coda_tensor_t* dst, void* stream);

/* Data-parallel weight gradient with its cross-rank sum fused into the GEMM epilogue
 * (B200 extension; replaces "wgrad GEMM, then NCCL all-reduce" for the weight gradients
 * the token-sharded block sums over ranks, reference kernels.py:936-1001).  Every rank
 * launches the same problem (its own token shard as K).  Output tile t is owned by rank
 * t % world: each rank dumps its f32 partial of t into slots[owner] (peer memory, e.g.
 * CUDA IPC over NVLink), then arrives on counters[owner]; the last of the world arrivals
 * sums the partials in rank order (bitwise deterministic, independent of arrival order),
 * rounds to bf16 once -- the reference's single store rounding, engine.py:443-447 -- and
 * writes the tile into out[r] of every rank.  Nothing waits on another rank, so ranks need
 * no co-scheduling; out[] is complete on all ranks once every rank's launch has finished
 * (the caller's cross-rank barrier).  Counters must be zero before the first launch and
 * are left zero; slot and counter buffers may be reused by the next launch only after
 * that barrier.  Sizes per rank: coda_peer_reduce_sizes. */
typedef struct {
    int32_t  world;                      /* ranks, 1 .. CODA_MAX_PEERS */
    int32_t  rank;                       /* this rank */
    void*    slots[CODA_MAX_PEERS];      /* per rank: f32 landing buffer (slot_bytes) */
    int32_t* counters[CODA_MAX_PEERS];   /* per rank: arrival counters (counter_bytes) */
    void*    out[CODA_MAX_PEERS];        /* per rank: bf16 (m, n) result, row stride ld_out */
    int64_t  ld_out;
    int64_t  slot_bytes;                 /* size of every rank's slots / counters buffer */
    int64_t  counter_bytes;
} coda_peer_reduce_t;

int coda_peer_reduce_sizes(int64_t m, int64_t n, int32_t world, int64_t* slot_bytes, int64_t* counter_bytes);

int coda_gemm_peer_reduce(const coda_problem_t* problem, const coda_tensor_t* a, const coda_tensor_t* b,
                          const coda_peer_reduce_t* peer, void* stream);

/* Engine schedule options (defaults from the environment); each variant computes
 * the same program: "pdl" 0/1 programmatic dependent launch, "cg" 1/2 CTA-pair
 * mainloop, "generic" 0/1 force the generic epilogue interpreter, "raster" >= 1
 * raster group, "split" 0/1 wave-tail split-K, "split_min_k" the smallest K that
 * is split (default 4096) and "split_piece_kb" the fewest 64-wide k-blocks per piece
 * (default 32) (splitting changes only the deterministic f32 accumulation order),
 * "st_tma" -1 / 0 / 1 the epilogue store path (-1 per launch: coalesced lane stores,
 * TMA stores for the SwiGLU backward with K < 4096; 0 / 1 force one; same bits).
 * Process-wide.  Measurement knobs ("ring", "prefetch", "ablate" — the last makes
 * results invalid) exist only in experiment builds (-DCODA_EXPERIMENTS) and return
 * CODA_E_CONFIG from the product library. */
int coda_set_option(const char* name, int value);

/* Number of SMs the persistent kernel sizes its grid for (0 if no device). */
int coda_num_sms(void);

/* Library build identifier, e.g. "coda sm_100a tcgen05". */
const char* coda_version(void);

/* Thread-local text of the last error. */
const char* coda_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CODA_H */
