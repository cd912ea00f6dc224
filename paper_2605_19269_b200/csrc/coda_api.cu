// coda_api.cu — extern "C" entry points declared in include/coda.h.
//
// Validation happens here, before anything is enqueued, and maps onto the
// reference error taxonomy (errors.py:9-56).  The library never allocates
// device memory; TMA descriptors are encoded on the host per launch (cached)
// and passed as __grid_constant__ kernel parameters.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <utility>

#include "../../include/coda.h"
#include "coda_aux.cuh"
#include "coda_gemm.cuh"
#include "coda_fast.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) return fail(CODA_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return CODA_OK;
}

int esize(int dtype) {
    switch (dtype) {
    case CODA_BF16: return 2;
    case CODA_F32: return 4;
    case CODA_I64: return 8;
    case CODA_I32: return 4;
    default: return 0;
    }
}

// Make the runtime's current device the one owning `ptr` (torch may run on any device)
// for the duration of one entry point; the caller's current device is restored when
// the guard goes out of scope, so nothing leaks into torch's current_device.
struct DeviceGuard {
    int prev = -1;
    int dev = -1;
    ~DeviceGuard() {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
};

int bind_device(const void* ptr, DeviceGuard& g) {
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(CODA_E_BINDING, "pointer %p is not a CUDA allocation", ptr);
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
        return fail(CODA_E_BINDING, "pointer %p is not device memory", ptr);
    int cur = -1;
    cudaGetDevice(&cur);
    g.prev = cur;
    g.dev = at.device;
    if (cur != at.device) {
        if (cudaSetDevice(at.device) != cudaSuccess) return fail(CODA_E_CUDA, "cudaSetDevice(%d) failed", at.device);
    }
    return CODA_OK;
}

int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

// Per-device one-time setup (function attributes are per device): bit d of `mask`.
constexpr int MAX_DEVICES = 64;
bool first_use_on_device(std::atomic<uint64_t>& mask) {
    const int d = current_device();
    if (d < 0 || d >= MAX_DEVICES) return true;
    const uint64_t bit = 1ull << d;
    return (mask.fetch_or(bit) & bit) == 0;
}

int check_tensor2d(const coda_tensor_t* t, const char* name, int dtype) {
    if (!t || !t->ptr) return fail(CODA_E_BINDING, "%s: null tensor", name);
    if (t->dtype != dtype) return fail(CODA_E_BINDING, "%s: dtype %d, expected %d", name, t->dtype, dtype);
    if (t->rows <= 0 || t->cols <= 0) return fail(CODA_E_DIMENSION, "%s: non-positive shape", name);
    const int es = esize(dtype);
    if ((reinterpret_cast<uintptr_t>(t->ptr) & 15) != 0)
        return fail(CODA_E_BINDING, "%s: base pointer must be 16-byte aligned", name);
    if (t->rows > 1 && ((t->ld * es) % 16 != 0 || t->ld < t->cols))
        return fail(CODA_E_BINDING, "%s: leading dimension %lld invalid (needs >= cols and 16-byte rows)",
                    name, (long long)t->ld);
    return CODA_OK;
}

// ---------------------------------------------------------------- TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

struct MapKey {
    const void* ptr;
    uint64_t d0, d1, stride;
    uint32_t b0, b1;
    int dtype, swz;
    bool operator==(const MapKey& o) const {
        return ptr == o.ptr && d0 == o.d0 && d1 == o.d1 && stride == o.stride && b0 == o.b0 && b1 == o.b1 &&
               dtype == o.dtype && swz == o.swz;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey& k) const {
        size_t h = std::hash<const void*>()(k.ptr);
        h ^= std::hash<uint64_t>()(k.d0 * 1315423911ull + k.d1) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
        h ^= std::hash<uint64_t>()(k.stride * 2654435761ull + k.b0 * 131 + k.b1 * 7 + k.dtype * 3 + k.swz) +
             (h << 6) + (h >> 2);
        return h;
    }
};

std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// 2-D tensor map, dim0 innermost (contiguous); swz = swizzle span in bytes (0/32/64/128).
int make_map(CUtensorMap* out, const void* ptr, uint64_t d0, uint64_t d1, uint64_t row_bytes, uint32_t b0,
             uint32_t b1, int dtype = CODA_BF16, int swz = 128) {
    MapKey key{ptr, d0, d1, row_bytes, b0, b1, dtype, swz};
    {
        std::lock_guard<std::mutex> lk(g_map_mu);
        auto it = g_maps.find(key);
        if (it != g_maps.end()) {
            *out = it->second;
            return CODA_OK;
        }
    }
    auto enc = get_encode();
    if (!enc) return fail(CODA_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {d0, d1};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {b0, b1};
    cuuint32_t es[2] = {1, 1};
    const CUtensorMapSwizzle sw = swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swz == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swz == 32  ? CU_TENSOR_MAP_SWIZZLE_32B
                                             : CU_TENSOR_MAP_SWIZZLE_NONE;
    const CUtensorMapDataType dt = dtype == CODA_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUresult r = enc(out, dt, 2, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(CODA_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 4096) g_maps.clear();
    g_maps.emplace(key, *out);
    return CODA_OK;
}

int num_sms() {
    static std::atomic<int> cache[MAX_DEVICES];   // 0 = not queried yet
    const int d = current_device();
    if (d >= 0 && d < MAX_DEVICES && cache[d].load() > 0) return cache[d].load();
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    if (d >= 0 && d < MAX_DEVICES && n > 0) cache[d].store(n);
    return n;
}

// SMs a launch may occupy: all of them, or the caller's cap (sm_limit > 0) so that
// a concurrent collective on another stream keeps SMs of its own.
int usable_sms(int sm_limit) {
    const int n = num_sms();
    return (sm_limit > 0 && sm_limit < n) ? sm_limit : n;
}

// ---------------------------------------------------------------- launches (PDL + clusters)
// Runtime options (environment defaults, overridable through coda_set_option so
// variants can be compared interleaved inside one process).  Product options change
// only the schedule: every variant computes the reference program (the wave-tail
// split changes f32 accumulation order, deterministically).  The measurement knobs
// (L2 prefetch, ring depth, epilogue ablations that make results invalid) exist only
// in experiment builds (-DCODA_EXPERIMENTS, _build.build(experiments=True) ->
// libcoda_exp.so, used by tools/); the product library rejects them.
struct Options {
    int pdl = 1;          // programmatic dependent launch
    int cg = 2;           // CTA-pair (2) or single-CTA (1) specialised kernels
    int generic = 0;      // force the generic epilogue interpreter
    int raster = 8;       // raster group (pair m-tiles)
    int split = 1;        // split the partial last wave along K
    // ... only for launches with at least this K, in pieces of at least split_piece_kb
    // 64-wide k-blocks (profiles/r02_session3/split_ab: 4096 / 32 vs the round-2 8192 / 4:
    // 4096^3 -1.5 %, 2048x28672x4096 -1.3 %, K10's shape -0.8 %, whole steps within noise)
    int split_min_k = 4096;
    int split_piece_kb = 32;
    int prefetch = 0;     // [experiments] L2 prefetch distance (k-blocks beyond the smem ring)
    int ablate = 0;       // [experiments] epilogue ablations (results invalid)
    int ring = 0;         // [experiments] operand ring stages in use (0 = the compiled depth)
    int rope_u = 0;       // [experiments] rope_backward_stat: 0 auto, 3 / 6 deep-load sweeps, 1 plain compact
    int persist = 1;      // [experiments] 0: one tile per cluster (non-persistent, hardware dispatch order)
    int wave_sync = 0;    // [experiments] soft wave barrier milestone in % of a tile's k-blocks (0 = off)
    int backoff = 0;      // [experiments] epilogue accumulator-wait sleep (ns)
    int st_tma = -1;      // staged epilogue stores: -1 per-launch choice, 0 lanes' copy-out, 1 TMA
    Options() {
        if (const char* e = getenv("CODA_PDL")) pdl = e[0] != '0';
        if (const char* e = getenv("CODA_CG")) cg = e[0] == '1' ? 1 : 2;
        if (const char* e = getenv("CODA_FORCE_GENERIC")) generic = e[0] && e[0] != '0';
        if (const char* e = getenv("CODA_RASTER_GROUP")) { const int g = atoi(e); if (g > 0) raster = g; }
        if (const char* e = getenv("CODA_SPLIT")) split = e[0] != '0';
#ifdef CODA_EXPERIMENTS
        if (const char* e = getenv("CODA_PREFETCH")) prefetch = atoi(e);
        if (const char* e = getenv("CODA_WAVE_SYNC")) wave_sync = atoi(e);
#endif
    }
};
Options& opts() {
    static Options o;
    return o;
}

bool pdl_enabled() { return opts().pdl != 0; }

// Launch with programmatic stream serialization (kernel N+1's prologue overlaps
// kernel N's tail; every kernel calls griddep_wait() before touching global
// memory) and an optional cluster shape.
template <typename... KArgs, typename... Args>
int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
               const char* what, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (pdl_enabled()) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (cluster > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = (unsigned)cluster;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), what);
}

template <typename TS>
int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const coda::GemmParams& P, cudaStream_t st,
                int sm_limit) {
    static std::atomic<uint64_t> configured{0};
    const size_t smem = coda::gemm_smem_bytes();
    if (first_use_on_device(configured)) {
        cudaError_t e = cudaFuncSetAttribute(coda::coda_gemm_kernel<TS>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(gemm smem)");
    }
    const int nsm = usable_sms(sm_limit);
    const int grid = P.ntiles < nsm ? P.ntiles : nsm;
    return launch_pdl(coda::coda_gemm_kernel<TS>, dim3(grid), dim3(coda::NUM_THREADS), smem, st, 1,
                      "coda_gemm_kernel launch", ma, mb, P);
}

inline unsigned grid1d(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }


// ---------------------------------------------------------------- specialised epilogues
using coda::F_AUX;
using coda::F_GATHER;
using coda::F_LSE;
using coda::F_OUT_F32;
using coda::F_PEER;
using coda::F_RESIDUAL;
using coda::F_RMSBWD;
using coda::F_RMSBWD_ACC;
using coda::F_ROPE;
using coda::F_ROWDOT;
using coda::F_ROWSCALE;
using coda::F_ROWVEC;
using coda::F_STORE_MAIN;
using coda::F_SUMSQ;
using coda::F_SWIGLU;
using coda::F_SWIGLU_BWD;
using coda::F_XENT_BWD;

#define CODA_FAST_SETS(X)                                             \
    X(F_STORE_MAIN)                                                   \
    X(F_STORE_MAIN | F_OUT_F32)                                       \
    X(F_ROPE | F_STORE_MAIN)                                          \
    X(F_SWIGLU | F_STORE_MAIN)                                        \
    X(F_AUX | F_SWIGLU | F_STORE_MAIN)                                \
    X(F_RESIDUAL | F_AUX | F_SUMSQ | F_ROWVEC | F_STORE_MAIN)         \
    X(F_RESIDUAL | F_AUX | F_SUMSQ)                                   \
    X(F_ROWSCALE | F_STORE_MAIN)                                      \
    X(F_ROWSCALE | F_AUX | F_SWIGLU | F_STORE_MAIN)                   \
    X(F_ROWSCALE | F_ROPE | F_STORE_MAIN)                             \
    X(F_RMSBWD | F_STORE_MAIN)                                        \
    X(F_RMSBWD | F_RMSBWD_ACC | F_STORE_MAIN)                         \
    X(F_SWIGLU_BWD | F_STORE_MAIN)                                    \
    X(F_SUMSQ | F_STORE_MAIN)                                         \
    X(F_RESIDUAL | F_STORE_MAIN)                                      \
    X(F_GATHER | F_LSE | F_STORE_MAIN)                                \
    X(F_GATHER | F_LSE)                                               \
    X(F_ROWSCALE | F_GATHER | F_LSE)                                  \
    X(F_ROWSCALE | F_GATHER | F_LSE | F_STORE_MAIN)                   \
    X(F_ROWDOT | F_ROWSCALE | F_STORE_MAIN)                           \
    X(F_ROWSCALE | F_XENT_BWD | F_STORE_MAIN)                         \
    X(F_ROWDOT | F_ROWSCALE | F_STORE_MAIN | F_OUT_F32)              \
    X(F_PEER)

template <int FL, int CG>
int launch_fast_fl(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mm, const CUtensorMap& mx,
                   const CUtensorMap& s0, const CUtensorMap& s1, const coda::FastParams& P, cudaStream_t st,
                   int units) {
    static std::atomic<uint64_t> configured{0};
    const size_t smem = coda::fast_smem_bytes<CG, FL>();
    auto kern = coda::coda_gemm_fast<__nv_bfloat16, FL, CG>;
    if (first_use_on_device(configured)) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(fast smem)");
        if (CG > 1) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
            if (e != cudaSuccess) cudaGetLastError();
        }
    }
    int grid = (P.mp.nitems < units ? P.mp.nitems : units) * CG;
#ifdef CODA_EXPERIMENTS
    if (opts().persist == 0 && P.mp.split <= 1) grid = P.mp.nitems * CG;   // one tile per cluster, hardware order
#endif
    return launch_pdl(kern, dim3((unsigned)grid), dim3(coda::FAST_THREADS), smem, st, CG, "coda_gemm_fast launch",
                      ma, mb, mm, mx, s0, s1, P);
}

int fast_cg() { return opts().cg; }

bool fast_supported(int fl) {
#define CODA_FAST_CASE(F) if (fl == (F)) return true;
    CODA_FAST_SETS(CODA_FAST_CASE)
#undef CODA_FAST_CASE
    return false;
}

int launch_fast(int fl, int cg, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mm,
                const CUtensorMap& mx, const CUtensorMap& s0, const CUtensorMap& s1, const coda::FastParams& P,
                cudaStream_t st, int units) {
#define CODA_FAST_CASE(F)                                                                \
    if (fl == (F))                                                                       \
        return cg == 2 ? launch_fast_fl<(F), 2>(ma, mb, mm, mx, s0, s1, P, st, units)    \
                       : launch_fast_fl<(F), 1>(ma, mb, mm, mx, s0, s1, P, st, units);
    CODA_FAST_SETS(CODA_FAST_CASE)
#undef CODA_FAST_CASE
    return fail(CODA_E_CONFIG, "no specialised kernel for flags 0x%x", fl);
}

// Raster group: m-tiles swept together across all n-tiles.  8 (pair) m-tiles was
// measured best on the C4 block (sweep 4/8/16/32/64, profiles/r01_raster_sweep.md);
// CODA_RASTER_GROUP overrides it for experiments.
int raster_group(int ntm, int tile_m, int64_t k) {
    (void)tile_m;
    (void)k;
    int g = opts().raster;
    if (g < 1) g = 1;
    if (g > ntm) g = ntm;
    return g;
}

// Map a validated program onto the flag set of a specialised kernel (or -1).
int match_fast(const coda_problem_t* pr, const coda_step_t* steps, int nsteps, const coda_store_t* stores) {
    if (opts().generic || pr->storage != CODA_BF16) return -1;
    int fl = 0, last_rank = 0;
    auto rank_ok = [&](int rk) {
        if (rk <= last_rank) return false;
        last_rank = rk;
        return true;
    };
    for (int s = 0; s < nsteps; ++s) {
        const coda_step_t& st = steps[s];
        if (st.width != 32) return -1;   // every fast op runs at factor 1
        switch (st.op) {
        case CODA_OP_PARTIAL_ROWDOT:
            if (!rank_ok(1) || !stores[st.arg[1]].aligned) return -1;
            fl |= F_ROWDOT; break;
        case CODA_OP_ROW_SCALE: if (!rank_ok(2)) return -1; fl |= F_ROWSCALE; break;
        case CODA_OP_RESIDUAL_ADD: if (!rank_ok(3)) return -1; fl |= F_RESIDUAL; break;
        case CODA_OP_AUX_TILE_STORE: if (!rank_ok(4)) return -1; fl |= F_AUX; break;
        case CODA_OP_PARTIAL_SUMSQ:
            if (!rank_ok(5) || !stores[st.arg[0]].aligned) return -1;
            fl |= F_SUMSQ; break;
        case CODA_OP_ROW_VEC_MUL: if (!rank_ok(6)) return -1; fl |= F_ROWVEC; break;
        case CODA_OP_ROPE: if (!rank_ok(7)) return -1; fl |= F_ROPE; break;
        case CODA_OP_TARGET_GATHER: if (!rank_ok(8)) return -1; fl |= F_GATHER; break;
        case CODA_OP_ONLINE_LSE:
            if (!rank_ok(9) || !stores[st.arg[0]].aligned) return -1;
            fl |= F_LSE; break;
        case CODA_OP_SWIGLU: if (!rank_ok(10)) return -1; fl |= F_SWIGLU; break;
        case CODA_OP_SWIGLU_BWD:
            if (!rank_ok(10) || !stores[st.arg[2]].aligned) return -1;
            fl |= F_SWIGLU_BWD; break;
        case CODA_OP_XENT_BWD:
            if (!rank_ok(10) || !stores[st.arg[2]].aligned) return -1;
            fl |= F_XENT_BWD; break;
        case CODA_OP_RMSNORM_BWD:
            if (!rank_ok(10) || !stores[st.arg[6]].aligned) return -1;
            fl |= F_RMSBWD | (st.arg[4] >= 0 ? F_RMSBWD_ACC : 0); break;
        default: return -1;
        }
    }
    if (pr->store_main) fl |= F_STORE_MAIN;
    if (pr->out_dtype == CODA_F32) {
        if (fl != F_STORE_MAIN && fl != (F_ROWDOT | F_ROWSCALE | F_STORE_MAIN)) return -1;
        fl |= F_OUT_F32;
    }
    return fast_supported(fl) ? fl : -1;
}

int store_swizzle(int row_bytes) { return row_bytes >= 128 ? 128 : row_bytes; }

}  // namespace

extern "C" {

const char* coda_last_error(void) { return g_err.c_str(); }

const char* coda_version(void) {
#ifdef CODA_EXPERIMENTS
    return "coda sm_100a tcgen05 2-CTA 256x256x64 persistent (experiments build)";
#else
    return "coda sm_100a tcgen05 2-CTA 256x256x64 persistent";
#endif
}

int coda_num_sms(void) { return num_sms(); }

int coda_set_option(const char* name, int value) {
    if (!name) return fail(CODA_E_BINDING, "null option name");
    const std::string n(name);
    if (n == "pdl") opts().pdl = value != 0;
    else if (n == "cg") {
        if (value != 1 && value != 2) return fail(CODA_E_CONFIG, "cg must be 1 or 2");
        opts().cg = value;
    } else if (n == "generic") opts().generic = value != 0;
    else if (n == "split") opts().split = value != 0;
    else if (n == "split_piece_kb") {
        if (value < 1) return fail(CODA_E_CONFIG, "split_piece_kb must be >= 1");
        opts().split_piece_kb = value;
    } else if (n == "split_min_k") {
        if (value < 0) return fail(CODA_E_CONFIG, "split_min_k must be >= 0");
        opts().split_min_k = value;
    } else if (n == "st_tma") {
        if (value < -1 || value > 1) return fail(CODA_E_CONFIG, "st_tma must be -1, 0 or 1");
        opts().st_tma = value;
    } else if (n == "raster") {
        if (value < 1) return fail(CODA_E_CONFIG, "raster group must be >= 1");
        opts().raster = value;
    }
#ifdef CODA_EXPERIMENTS
    else if (n == "ablate") opts().ablate = value;
    else if (n == "ring") opts().ring = value;
    else if (n == "rope_u") opts().rope_u = value;
    else if (n == "persist") opts().persist = value;
    else if (n == "wave_sync") opts().wave_sync = value;
    else if (n == "backoff") opts().backoff = value;
    else if (n == "prefetch") {
        if (value < 0 || value > 64) return fail(CODA_E_CONFIG, "prefetch distance must be in [0, 64]");
        opts().prefetch = value;
    }
#else
    else if (n == "ablate" || n == "ring" || n == "prefetch")
        return fail(CODA_E_CONFIG, "option %s exists only in experiment builds (-DCODA_EXPERIMENTS)", name);
#endif
    else return fail(CODA_E_CONFIG, "unknown option %s", name);
    return CODA_OK;
}

namespace {
int gemm_impl(const coda_problem_t* pr, const coda_tensor_t* a, const coda_tensor_t* b, const coda_step_t* steps,
              int nsteps, const coda_tensor_t* operands, int noperands, const coda_store_t* stores, int nstores,
              const coda_tensor_t* main_out, const coda_tensor_t* acc_in, void* stream,
              const coda_peer_reduce_t* peer);

int64_t peer_tiles(int64_t m, int64_t n) {
    const int64_t tile_m = (int64_t)coda::BM * fast_cg();
    return ((m + tile_m - 1) / tile_m) * ((n + coda::BN - 1) / coda::BN);
}
}  // namespace

int coda_peer_reduce_sizes(int64_t m, int64_t n, int32_t world, int64_t* slot_bytes, int64_t* counter_bytes) {
    if (m <= 0 || n <= 0) return fail(CODA_E_DIMENSION, "peer reduce: dims must be positive");
    if (world < 1 || world > CODA_MAX_PEERS) return fail(CODA_E_CONFIG, "peer reduce: world must be 1..%d", CODA_MAX_PEERS);
    if (!slot_bytes || !counter_bytes) return fail(CODA_E_BINDING, "peer reduce: null size outputs");
    const int64_t owned = (peer_tiles(m, n) + world - 1) / world;
    *slot_bytes = owned * world * fast_cg() * coda::BM * coda::BN * 4;
    *counter_bytes = owned * fast_cg() * 4;
    return 0;
}

int coda_gemm_peer_reduce(const coda_problem_t* problem, const coda_tensor_t* a, const coda_tensor_t* b,
                          const coda_peer_reduce_t* peer, void* stream) {
    if (!problem || !peer) return fail(CODA_E_BINDING, "null problem or peer descriptor");
    if (problem->storage != CODA_BF16) return fail(CODA_E_CONFIG, "peer reduce: storage must be bf16");
    if (opts().generic) return fail(CODA_E_CONFIG, "peer reduce runs on the specialised kernels only");
    int64_t need_slots = 0, need_ctr = 0;
    int rc = coda_peer_reduce_sizes(problem->m, problem->n, peer->world, &need_slots, &need_ctr);
    if (rc) return rc;
    if (peer->rank < 0 || peer->rank >= peer->world) return fail(CODA_E_CONFIG, "peer reduce: bad rank %d", peer->rank);
    if (peer->slot_bytes < need_slots || peer->counter_bytes < need_ctr)
        return fail(CODA_E_BINDING, "peer reduce: buffers too small (%lld / %lld bytes, need %lld / %lld)",
                    (long long)peer->slot_bytes, (long long)peer->counter_bytes, (long long)need_slots,
                    (long long)need_ctr);
    if (peer->ld_out < problem->n) return fail(CODA_E_DIMENSION, "peer reduce: ld_out < n");
    for (int r = 0; r < peer->world; ++r)
        if (!peer->slots[r] || !peer->counters[r] || !peer->out[r])
            return fail(CODA_E_BINDING, "peer reduce: null buffer for rank %d", r);
    coda_problem_t pr = *problem;
    pr.store_main = 0;
    pr.out_dtype = CODA_BF16;
    pr.workspace = nullptr;      // no wave-tail split: every tile is one rank's partial
    pr.workspace_bytes = 0;
    return gemm_impl(&pr, a, b, nullptr, 0, nullptr, 0, nullptr, 0, nullptr, nullptr, stream, peer);
}

int coda_gemm_epilogue(const coda_problem_t* pr, const coda_tensor_t* a, const coda_tensor_t* b,
                       const coda_step_t* steps, int nsteps, const coda_tensor_t* operands, int noperands,
                       const coda_store_t* stores, int nstores, const coda_tensor_t* main_out,
                       const coda_tensor_t* acc_in, void* stream) {
    return gemm_impl(pr, a, b, steps, nsteps, operands, noperands, stores, nstores, main_out, acc_in, stream, nullptr);
}

namespace {
int gemm_impl(const coda_problem_t* pr, const coda_tensor_t* a, const coda_tensor_t* b, const coda_step_t* steps,
              int nsteps, const coda_tensor_t* operands, int noperands, const coda_store_t* stores, int nstores,
              const coda_tensor_t* main_out, const coda_tensor_t* acc_in, void* stream,
              const coda_peer_reduce_t* peer) {
    if (!pr) return fail(CODA_E_BINDING, "null problem");
    const int64_t M = pr->m, N = pr->n, K = pr->k;
    if (M <= 0 || N <= 0 || K <= 0) return fail(CODA_E_DIMENSION, "problem dims must be positive");
    if (M > INT32_MAX / 2 || N > INT32_MAX / 4 || K > INT32_MAX / 2) return fail(CODA_E_DIMENSION, "problem too large");
    if (pr->storage != CODA_BF16 && pr->storage != CODA_F32)
        return fail(CODA_E_CONFIG, "storage dtype must be bf16 or f32");
    int rc;
    if ((rc = check_tensor2d(a, "a", CODA_BF16))) return rc;
    if ((rc = check_tensor2d(b, "b", CODA_BF16))) return rc;
    const int64_t ar = pr->trans_a ? K : M, ac = pr->trans_a ? M : K;
    const int64_t br = pr->trans_b ? N : K, bc = pr->trans_b ? K : N;
    if (a->rows != ar || a->cols != ac)
        return fail(CODA_E_DIMENSION, "a has shape (%lld,%lld), problem wants (%lld,%lld)", (long long)a->rows,
                    (long long)a->cols, (long long)ar, (long long)ac);
    if (b->rows != br || b->cols != bc)
        return fail(CODA_E_DIMENSION, "b has shape (%lld,%lld), problem wants (%lld,%lld)", (long long)b->rows,
                    (long long)b->cols, (long long)br, (long long)bc);
    if (nsteps < 0 || nsteps > CODA_MAX_STEPS) return fail(CODA_E_PROGRAM, "too many program steps (%d)", nsteps);
    if (noperands < 0 || noperands > CODA_MAX_OPERANDS || nstores < 0 || nstores > CODA_MAX_STORES)
        return fail(CODA_E_PROGRAM, "too many operands/stores");
    DeviceGuard dg;
    if ((rc = bind_device(a->ptr, dg))) return rc;

    coda::GemmParams P;
    memset(&P, 0, sizeof(P));
    P.M = (int)M;
    P.N = (int)N;
    P.K = (int)K;
    P.ntm = (int)((M + coda::BM - 1) / coda::BM);
    P.ntn = (int)((N + coda::BN - 1) / coda::BN);
    P.nk = (int)((K + coda::BK - 1) / coda::BK);
    P.ntiles = P.ntm * P.ntn;
    P.a_mn = pr->trans_a ? 1 : 0;
    P.b_mn = pr->trans_b ? 0 : 1;
    P.nsteps = nsteps;
    P.store_main = pr->store_main ? 1 : 0;
    P.out_f32 = pr->out_dtype == CODA_F32 ? 1 : 0;

    const int sdt = pr->storage;
    bool fin_source[CODA_MAX_OPERANDS] = {};
    int w = 32;
    for (int s = 0; s < nsteps; ++s) {
        const coda_step_t& cs = steps[s];
        coda::DevStep& d = P.steps[s];
        d.op = cs.op;
        d.w = cs.width;
        for (int i = 0; i < 7; ++i) d.a[i] = cs.arg[i];
        d.fin_src = cs.fin_src;
        d.fin_kind = cs.fin_kind;
        d.fin_d = cs.fin_d;
        d.fin_eps = cs.fin_eps;
        if (cs.fin_src != 0) {
            const int fs = cs.fin_src - 1;
            if (cs.op != CODA_OP_ROW_SCALE && cs.op != CODA_OP_RMSNORM_BWD)
                return fail(CODA_E_PROGRAM, "step %d: deferred finalizers apply to RowScale / RmsNormBackwardLocal", s);
            if (fs < 0 || fs >= noperands) return fail(CODA_E_PROGRAM, "step %d: bad finalizer source slot", s);
            const coda_tensor_t& t = operands[fs];
            if (t.dtype != CODA_F32 || t.rows != M || t.cols <= 0 || !t.ptr)
                return fail(CODA_E_BINDING, "step %d: finalizer source must be f32 (m, nb) partials", s);
            if (cs.fin_kind != CODA_FIN_RMS && cs.fin_kind != CODA_FIN_ROWDOT)
                return fail(CODA_E_PROGRAM, "step %d: unknown finalizer kind %d", s, cs.fin_kind);
            if (cs.fin_d <= 0) return fail(CODA_E_DEGENERATE, "step %d: finalizer width must be positive", s);
            fin_source[fs] = true;
        }
        if (d.w != w) return fail(CODA_E_PROGRAM, "step %d: width %d does not match running width %d", s, d.w, w);
        auto opnd_ok = [&](int i) { return i >= 0 && i < noperands; };
        auto stream_ok = [&](int i) { return i >= 0 && i < coda::MAX_ROW_STREAMS; };
        auto store_ok = [&](int i) { return i >= 0 && i < nstores; };
        bool ok = true;
        switch (cs.op) {
        case CODA_OP_ROW_VEC_MUL: case CODA_OP_ROW_SCALE: case CODA_OP_RESIDUAL_ADD: ok = opnd_ok(cs.arg[0]); break;
        case CODA_OP_AUX_TILE_STORE: case CODA_OP_PARTIAL_COLSUM: ok = store_ok(cs.arg[0]); break;
        case CODA_OP_PARTIAL_SUMSQ: case CODA_OP_ONLINE_LSE:
            ok = store_ok(cs.arg[0]) && w == 32 && stream_ok(cs.arg[6]); break;
        case CODA_OP_PARTIAL_ROWDOT:
            ok = opnd_ok(cs.arg[0]) && store_ok(cs.arg[1]) && w == 32 && stream_ok(cs.arg[6]); break;
        case CODA_OP_TARGET_GATHER: ok = opnd_ok(cs.arg[0]) && store_ok(cs.arg[1]) && w == 32; break;
        case CODA_OP_ROPE:
            ok = opnd_ok(cs.arg[0]) && opnd_ok(cs.arg[1]) && w >= 2;
            if (ok && cs.arg[3] > 0) {   // compact tables: arg3/arg4 = 1 + operand slot, arg5 = q-span width h
                const int h = cs.arg[5];
                // packed qkv (2h <= N: q and k share the h/2 angles, the rest is identity) or
                // a plain table over the whole width (h == N: column c takes angle c / 2)
                ok = opnd_ok(cs.arg[3] - 1) && opnd_ok(cs.arg[4] - 1) && h > 0 && h % 32 == 0 &&
                     (2 * (int64_t)h <= N || (int64_t)h == N);
                for (int j = 3; ok && j <= 4; ++j) {
                    const coda_tensor_t& t = operands[cs.arg[j] - 1];
                    ok = t.dtype == CODA_BF16 && t.rows == M && t.cols == h / 2;
                }
                if (!ok) return fail(CODA_E_BINDING, "step %d: compact RoPE tables must be bf16 (m, h/2), h %% 32 == 0, 2h <= n or h == n", s);
            }
            break;
        case CODA_OP_SWIGLU:
            if (w < 2) return fail(CODA_E_CONFIG, "GPU epilogue supports running width factors 1/32 .. 2");
            w /= 2; break;
        case CODA_OP_SWIGLU_BWD:
            ok = opnd_ok(cs.arg[0]) && store_ok(cs.arg[1]) && store_ok(cs.arg[2]) && w == 32 &&
                 stream_ok(cs.arg[6]);
            w = 64; break;
        case CODA_OP_XENT_BWD:
            ok = opnd_ok(cs.arg[0]) && opnd_ok(cs.arg[1]) && store_ok(cs.arg[2]) && w == 32 && stream_ok(cs.arg[6]);
            break;
        case CODA_OP_RMSNORM_BWD:
            ok = opnd_ok(cs.arg[0]) && opnd_ok(cs.arg[1]) && opnd_ok(cs.arg[2]) && opnd_ok(cs.arg[3]) &&
                 (cs.arg[4] == -1 || opnd_ok(cs.arg[4])) && store_ok(cs.arg[5]) && store_ok(cs.arg[6]) && w == 32;
            break;
        default: return fail(CODA_E_PROGRAM, "step %d: unknown op %d", s, cs.op);
        }
        if (!ok) return fail(CODA_E_PROGRAM, "step %d (op %d): bad slot index or width", s, cs.op);
    }
    P.out_w = w;
    for (int i = 0; i < noperands; ++i) {
        const coda_tensor_t& t = operands[i];
        if (!t.ptr) return fail(CODA_E_BINDING, "operand %d is null", i);
        if (t.rows > 1 && t.dtype == sdt && !fin_source[i]) {
            char nm[32];
            snprintf(nm, sizeof(nm), "operand %d", i);
            if ((rc = check_tensor2d(&t, nm, sdt))) return rc;
            if (t.rows != M) return fail(CODA_E_DIMENSION, "operand %d has %lld rows, expected %lld", i,
                                         (long long)t.rows, (long long)M);
        }
        P.opnd[i].ptr = t.ptr;
        P.opnd[i].ld = t.ld;
        P.opnd[i].cols = t.cols;
    }
    for (int i = 0; i < nstores; ++i) {
        const coda_store_t& s = stores[i];
        if (!s.t.ptr) return fail(CODA_E_BINDING, "store %d is null", i);
        if (s.kind == 0) {
            char nm[32];
            snprintf(nm, sizeof(nm), "store %d", i);
            if ((rc = check_tensor2d(&s.t, nm, sdt))) return rc;
        } else if (s.kind >= 1 && s.kind <= 3 && !s.piece_map) {
            return fail(CODA_E_BINDING, "store %d needs a piece map", i);
        }
        P.store[i].ptr = s.t.ptr;
        P.store[i].ld = s.t.ld;
        P.store[i].cols = s.t.cols;
        P.store[i].map = s.piece_map;
    }
    if (P.store_main) {
        const int odt = P.out_f32 ? CODA_F32 : CODA_BF16;
        if ((rc = check_tensor2d(main_out, "main", odt))) return rc;
        const int64_t want = N * w / 32;
        if (main_out->rows != M || main_out->cols != want)
            return fail(CODA_E_DIMENSION, "main output has shape (%lld,%lld), expected (%lld,%lld)",
                        (long long)main_out->rows, (long long)main_out->cols, (long long)M, (long long)want);
        P.out = main_out->ptr;
        P.ld_out = main_out->ld;
    }

    if (acc_in) {
        if ((rc = check_tensor2d(acc_in, "acc_in", CODA_F32))) return rc;
        if (acc_in->rows != M || acc_in->cols != N)
            return fail(CODA_E_DIMENSION, "acc_in has shape (%lld,%lld), expected (%lld,%lld)",
                        (long long)acc_in->rows, (long long)acc_in->cols, (long long)M, (long long)N);
        P.acc_in = static_cast<const float*>(acc_in->ptr);
        P.ld_acc = acc_in->ld;
    }

    CUtensorMap ma, mb;
    if (!pr->trans_a) rc = make_map(&ma, a->ptr, (uint64_t)K, (uint64_t)M, (uint64_t)a->ld * 2, coda::BK, coda::BM);
    else rc = make_map(&ma, a->ptr, (uint64_t)M, (uint64_t)K, (uint64_t)a->ld * 2, 64, coda::BK);
    if (rc) return rc;
    if (pr->trans_b) rc = make_map(&mb, b->ptr, (uint64_t)K, (uint64_t)N, (uint64_t)b->ld * 2, coda::BK, coda::BN);
    else rc = make_map(&mb, b->ptr, (uint64_t)N, (uint64_t)K, (uint64_t)b->ld * 2, 64, coda::BK);
    if (rc) return rc;

    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);

    const int fl = peer ? (int)coda::F_PEER : match_fast(pr, steps, nsteps, stores);
    if (fl >= 0) {
        const int cg = fast_cg();
        coda::FastParams F;
        memset(&F, 0, sizeof(F));
        const int tile_m = coda::BM * cg;
        const int ntm = (int)((M + tile_m - 1) / tile_m);
        const int ntiles = ntm * P.ntn;
        F.mp = coda::MainParams{P.M, P.N, P.K, ntm, P.ntn, P.nk, ntiles, P.a_mn, P.b_mn,
                                raster_group(ntm, tile_m, K), ntiles, 0, 1, ntiles, opts().prefetch, opts().ring};
        // wave-tail split: the r tiles of the partial last wave run as s K-pieces each
        const int units = std::max(1, usable_sms(pr->sm_limit) / cg);
        const int r = units > 0 ? ntiles % units : 0;
        // only long-K launches: the dump / fixed-order fold costs ~10-20 us, which a split of a
        // short mainloop cannot repay (tools/gemm_bench.py: +9 % at K=16384, -8 % at K=4096)
        if (!peer && opts().split && r > 0 && K >= opts().split_min_k && pr->workspace &&
            pr->workspace_bytes > (64 << 10)) {
            int sp = units / r;
            if (sp > P.nk / opts().split_piece_kb) sp = P.nk / opts().split_piece_kb;
            if (sp > 16) sp = 16;
            const int64_t tile_bytes = (int64_t)cg * coda::BM * coda::BN * 4;
            // every piece dumps its partial tile; one arrival counter per (tail tile, rank, warp)
            while (sp >= 2 && (int64_t)r * sp * tile_bytes > pr->workspace_bytes - (64 << 10)) --sp;
            if ((int64_t)r * cg * 4 > (32 << 10)) sp = 0;   // one arrival counter per (tail tile, rank)
            if (sp >= 2) {
                F.mp.full_tiles = ntiles - r;
                F.mp.tail = r;
                F.mp.split = sp;
                F.mp.nitems = ntiles - r + r * sp;
                F.flags = static_cast<int*>(pr->workspace);
                F.ws = reinterpret_cast<float*>(static_cast<char*>(pr->workspace) + (64 << 10));
            }
        }
#ifdef CODA_EXPERIMENTS
        // soft wave barrier: counters live in the second half of the workspace's counter region
        if (opts().wave_sync > 0 && pr->workspace && K >= opts().split_min_k) {
            const int nw = (F.mp.nitems + units - 1) / units;
            if ((nw + 1) * 4 <= (32 << 10)) {
                F.mp.wave_pct = opts().wave_sync;
                F.mp.wave_ctr = reinterpret_cast<int*>(static_cast<char*>(pr->workspace) + (32 << 10));
            }
        }
#endif
        if (peer) {
            F.peer_world = peer->world;
            F.peer_rank = peer->rank;
            for (int r = 0; r < peer->world; ++r) {
                F.peer_slots[r] = static_cast<float*>(peer->slots[r]);
                F.peer_ctr[r] = peer->counters[r];
                F.peer_out[r] = static_cast<__nv_bfloat16*>(peer->out[r]);
            }
            F.ld_peer_out = peer->ld_out;
        }
        F.acc_in = P.acc_in;
        F.ld_acc = P.ld_acc;
        F.ablate = opts().ablate;
        F.backoff = opts().backoff;
        // epilogue store path: the lanes' coalesced copy-out, except the SwiGLU backward
        // (three boxes per chunk) on a short mainloop, where the TMA engine is cheaper
        F.st_tma = opts().st_tma >= 0 ? opts().st_tma : ((fl & coda::F_SWIGLU_BWD) && K < 4096 ? 1 : 0);
        F.rope_sign = 1.0f;
        const void* rope_c = nullptr;
        const void* rope_s = nullptr;
        int64_t ld_rope_c = 0, ld_rope_s = 0;
        int aux_slot = -1;
        for (int s = 0; s < nsteps; ++s) {
            const coda_step_t& cs = steps[s];
            const coda::DevOperand* o = P.opnd;
            switch (cs.op) {
            case CODA_OP_ROW_SCALE:
                F.rowscale = (const float*)o[cs.arg[0]].ptr;
                if (cs.fin_src) {
                    const coda::DevOperand& fp = o[cs.fin_src - 1];
                    F.rs_fin = (const float*)fp.ptr; F.ld_rs_fin = fp.ld; F.rs_fin_nb = (int)fp.cols;
                    F.rs_fin_kind = cs.fin_kind; F.rs_fin_d = (float)cs.fin_d; F.rs_fin_eps = cs.fin_eps;
                }
                break;
            case CODA_OP_PARTIAL_ROWDOT:
                F.rowdot_x = o[cs.arg[0]].ptr; F.ld_rowdot_x = o[cs.arg[0]].ld;
                F.rowpart = (float*)P.store[cs.arg[1]].ptr; F.ld_rowpart = P.store[cs.arg[1]].ld;
                F.rowpart_map = P.store[cs.arg[1]].map; break;
            case CODA_OP_RESIDUAL_ADD: F.residual = o[cs.arg[0]].ptr; F.ld_res = o[cs.arg[0]].ld; break;
            case CODA_OP_AUX_TILE_STORE: aux_slot = cs.arg[0]; break;
            case CODA_OP_PARTIAL_SUMSQ:
                F.rowpart = (float*)P.store[cs.arg[0]].ptr; F.ld_rowpart = P.store[cs.arg[0]].ld;
                F.rowpart_map = P.store[cs.arg[0]].map; break;
            case CODA_OP_ROW_VEC_MUL: F.rowvec = (const float*)o[cs.arg[0]].ptr; break;
            case CODA_OP_TARGET_GATHER:
                F.labels = (const int64_t*)o[cs.arg[0]].ptr;
                F.target = (float*)P.store[cs.arg[1]].ptr; break;
            case CODA_OP_XENT_BWD:
                F.xent_lse = (const float*)o[cs.arg[0]].ptr;
                F.labels = (const int64_t*)o[cs.arg[1]].ptr;
                memcpy(&F.xent_scale, &cs.arg[3], sizeof(float));
                F.rowpart = (float*)P.store[cs.arg[2]].ptr; F.ld_rowpart = P.store[cs.arg[2]].ld;
                F.rowpart_map = P.store[cs.arg[2]].map; break;
            case CODA_OP_ONLINE_LSE:
                F.rowpart = (float*)P.store[cs.arg[0]].ptr; F.ld_rowpart = P.store[cs.arg[0]].ld;
                F.rowpart_map = P.store[cs.arg[0]].map; break;
            case CODA_OP_ROPE:
                F.cosp = o[cs.arg[0]].ptr; F.ld_cos = o[cs.arg[0]].ld;
                F.sinp = o[cs.arg[1]].ptr; F.ld_sin = o[cs.arg[1]].ld;
                F.rope_sign = cs.arg[2] ? -1.0f : 1.0f;
                if (cs.arg[3] > 0) {
                    rope_c = o[cs.arg[3] - 1].ptr; ld_rope_c = o[cs.arg[3] - 1].ld;
                    rope_s = o[cs.arg[4] - 1].ptr; ld_rope_s = o[cs.arg[4] - 1].ld;
                    F.rope_h = cs.arg[5];
                }
                break;
            case CODA_OP_SWIGLU_BWD:
                F.preact2 = o[cs.arg[0]].ptr; F.ld_pre2 = o[cs.arg[0]].ld;
                aux_slot = cs.arg[1];
                F.rowpart = (float*)P.store[cs.arg[2]].ptr; F.ld_rowpart = P.store[cs.arg[2]].ld;
                F.rowpart_map = P.store[cs.arg[2]].map; break;
            case CODA_OP_RMSNORM_BWD:
                F.pre = o[cs.arg[0]].ptr; F.ld_pre = o[cs.arg[0]].ld;
                F.inv_rms = (const float*)o[cs.arg[1]].ptr;
                F.gamma = (const float*)o[cs.arg[2]].ptr;
                F.stat = (const float*)o[cs.arg[3]].ptr;
                if (cs.fin_src) {
                    const coda::DevOperand& fp = o[cs.fin_src - 1];
                    F.st_fin = (const float*)fp.ptr; F.ld_st_fin = fp.ld; F.st_fin_nb = (int)fp.cols;
                    F.st_fin_kind = cs.fin_kind; F.st_fin_d = (float)cs.fin_d; F.st_fin_eps = cs.fin_eps;
                }
                if (cs.arg[4] >= 0) { F.grad_in = o[cs.arg[4]].ptr; F.ld_gin = o[cs.arg[4]].ld; }
                aux_slot = cs.arg[5];
                F.colpart = (float*)P.store[cs.arg[6]].ptr; F.ld_colpart = P.store[cs.arg[6]].ld;
                F.colpart_map = P.store[cs.arg[6]].map; break;
            default: break;
            }
        }
        CUtensorMap mm, mx;
        memset(&mm, 0, sizeof(mm));
        memset(&mx, 0, sizeof(mx));
        if (P.store_main) {
            const int odt = P.out_f32 ? CODA_F32 : CODA_BF16;
            const int es = P.out_f32 ? 4 : 2;
            const int wv = w;                  // values per 32-column chunk after the program
            const int rb = wv * es;
            // 128-byte rows are stored as two 64-byte-wide halves (coda_fast.cuh staged_store)
            const int bw = rb >= 128 ? wv / 2 : wv;
            rc = make_map(&mm, main_out->ptr, (uint64_t)main_out->cols, (uint64_t)M, (uint64_t)main_out->ld * es,
                          (uint32_t)bw, 32u, odt, store_swizzle(bw * es));
            if (rc) return rc;
            F.st_main = main_out->ptr; F.st_main_ld = main_out->ld * es; F.st_main_cols = main_out->cols * es;
        }
        if (aux_slot >= 0) {
            const coda_store_t& xs = stores[aux_slot];
            rc = make_map(&mx, xs.t.ptr, (uint64_t)xs.t.cols, (uint64_t)M, (uint64_t)xs.t.ld * 2, 32u, 32u, CODA_BF16,
                          64);
            if (rc) return rc;
            F.st_aux = xs.t.ptr; F.st_aux_ld = xs.t.ld * 2; F.st_aux_cols = xs.t.cols * 2;
        }
        if (cg == 2 && pr->trans_b) {   // K-major B box covers this CTA's 128-column half
            rc = make_map(&mb, b->ptr, (uint64_t)K, (uint64_t)N, (uint64_t)b->ld * 2, coda::BK, coda::BN / 2);
            if (rc) return rc;
        }
        // side-operand maps: 32-row boxes of one 32-column chunk (preact: 64 columns)
        CUtensorMap s0, s1;
        memset(&s0, 0, sizeof(s0));
        memset(&s1, 0, sizeof(s1));
        auto side_map = [&](CUtensorMap* out, const void* ptr, int64_t ld, int64_t cols, int box_cols) {
            return make_map(out, ptr, (uint64_t)cols, (uint64_t)M, (uint64_t)ld * 2, (uint32_t)box_cols, 32u,
                            CODA_BF16, box_cols * 2);
        };
        if (fl & F_RESIDUAL) rc = side_map(&s0, F.residual, F.ld_res, N, 32);
        if (!rc && (fl & F_ROWDOT)) rc = side_map(&s0, F.rowdot_x, F.ld_rowdot_x, N, 32);
        if (!rc && (fl & F_ROPE)) {
            if (F.rope_h > 0) {   // compact: 32 rows x 16 angles (32 B, SWIZZLE_32B)
                rc = side_map(&s0, rope_c, ld_rope_c, F.rope_h / 2, 16);
                if (!rc) rc = side_map(&s1, rope_s, ld_rope_s, F.rope_h / 2, 16);
            } else {
                rc = side_map(&s0, F.cosp, F.ld_cos, N, 32);
                if (!rc) rc = side_map(&s1, F.sinp, F.ld_sin, N, 32);
            }
        }
        if (!rc && (fl & F_SWIGLU_BWD)) rc = side_map(&s0, F.preact2, F.ld_pre2, 2 * N, 64);
        if (!rc && (fl & F_RMSBWD)) {
            rc = side_map(&s0, F.pre, F.ld_pre, N, 32);
            if (!rc && (fl & F_RMSBWD_ACC)) rc = side_map(&s1, F.grad_in, F.ld_gin, N, 32);
        }
        if (rc) return rc;
        return launch_fast(fl, cg, ma, mb, mm, mx, s0, s1, F, st, units);
    }
    if (sdt == CODA_BF16) return launch_gemm<__nv_bfloat16>(ma, mb, P, st, pr->sm_limit);
    return launch_gemm<float>(ma, mb, P, st, pr->sm_limit);
}
}  // namespace

int coda_finalize_rms(const float* p, int64_t m, int64_t nb, int64_t ld, int64_t d, float eps, float* r,
                      void* stream) {
    if (m <= 0 || nb <= 0) return fail(CODA_E_DIMENSION, "finalize_rms: empty partials");
    if (d <= 0) return fail(CODA_E_DEGENERATE, "partial blocks cover no columns");
    int rc;
    DeviceGuard dg;
    if ((rc = bind_device(p, dg))) return rc;
    if (nb <= 1024) {
        static std::atomic<uint64_t> cfg_done{0};
        if (first_use_on_device(cfg_done)) {
            cudaFuncSetAttribute(coda::coda_finalize_rms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
        }
        const size_t smem = (size_t)coda::FIN_ROWS * (nb + 1) * 4;
        return launch_pdl(coda::coda_finalize_rms_kernel, dim3((unsigned)((m + coda::FIN_ROWS - 1) / coda::FIN_ROWS)),
                          dim3(256), smem, (cudaStream_t)stream, 1, "finalize_rms", p, m, nb, ld, (float)d, eps, r);
    }
    return launch_pdl(coda::coda_finalize_rms_wide_kernel, dim3(grid1d(m, 256)), dim3(256), 0, (cudaStream_t)stream, 1,
                      "finalize_rms_wide", p, m, nb, ld, (float)d, eps, r);
}

int coda_finalize_rowdot(const float* p, int64_t m, int64_t nb, int64_t ld, int64_t d, float* s, void* stream) {
    if (m <= 0 || nb <= 0) return fail(CODA_E_DIMENSION, "finalize_rowdot: empty partials");
    if (d <= 0) return fail(CODA_E_CONFIG, "normalized width must be positive, got %lld", (long long)d);
    int rc;
    DeviceGuard dg;
    if ((rc = bind_device(p, dg))) return rc;
    if (nb <= 1024) {
        static std::atomic<uint64_t> cfg_done{0};
        if (first_use_on_device(cfg_done)) {
            cudaFuncSetAttribute(coda::coda_finalize_rowdot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 140 * 1024);
        }
        const size_t smem = (size_t)coda::FIN_ROWS * (nb + 1) * 4;
        return launch_pdl(coda::coda_finalize_rowdot_kernel, dim3((unsigned)((m + coda::FIN_ROWS - 1) / coda::FIN_ROWS)),
                          dim3(256), smem, (cudaStream_t)stream, 1, "finalize_rowdot", p, m, nb, ld, (float)d, s);
    }
    return launch_pdl(coda::coda_finalize_rowdot_wide_kernel, dim3(grid1d(m, 256)), dim3(256), 0, (cudaStream_t)stream,
                      1, "finalize_rowdot_wide", p, m, nb, ld, (float)d, s);
}

int coda_reduce_row_partials(const float* p, int64_t tm, int64_t n, int64_t ld, float* out, void* stream) {
    if (tm <= 0 || n <= 0) return fail(CODA_E_DIMENSION, "reduce_row_partials: empty partials");
    int rc;
    DeviceGuard dg;
    if ((rc = bind_device(p, dg))) return rc;
    return launch_pdl(coda::coda_reduce_row_partials_kernel, dim3(grid1d(n, 64)), dim3(64), 0, (cudaStream_t)stream, 1, "coda::coda_reduce_row_partials_kernel",
        p, tm, n, ld, out);
}

int coda_combine_lse(const float* p, int64_t m, int64_t nb, int64_t ld, float* lse, void* stream) {
    if (m <= 0 || nb <= 0) return fail(CODA_E_DIMENSION, "combine_lse: empty partials");
    int rc;
    DeviceGuard dg;
    if ((rc = bind_device(p, dg))) return rc;
    return launch_pdl(coda::coda_combine_lse_kernel, dim3(grid1d(m, 64)), dim3(64), 0, (cudaStream_t)stream, 1, "coda::coda_combine_lse_kernel",
        p, m, nb, ld, lse);
}

int coda_cross_entropy_finalize(const float* target, const float* lse, int64_t m, float* losses, void* stream) {
    if (m <= 0) return fail(CODA_E_DIMENSION, "cross_entropy_finalize: empty");
    int rc;
    DeviceGuard dg;
    if ((rc = bind_device(lse, dg))) return rc;
    return launch_pdl(coda::coda_ce_finalize_kernel, dim3(grid1d(m, 256)), dim3(256), 0, (cudaStream_t)stream, 1, "coda::coda_ce_finalize_kernel",
        target, lse, m, losses);
}

int coda_rope_backward_stat_compact(const coda_tensor_t* grad, const coda_tensor_t* rotated,
                                    const coda_tensor_t* cos_c, const coda_tensor_t* sin_c, int64_t h,
                                    coda_tensor_t* grad_z, float* rowdot, int64_t ld_rowdot, void* stream) {
    if (!grad || !rotated || !cos_c || !sin_c || !grad_z || !rowdot)
        return fail(CODA_E_BINDING, "rope_backward_stat_compact: null argument");
    int rc;
    const coda_tensor_t* ts[3] = {grad, rotated, grad_z};
    const char* nm[3] = {"grad", "rotated", "grad_z"};
    for (int i = 0; i < 3; ++i) {
        if ((rc = check_tensor2d(ts[i], nm[i], CODA_BF16))) return rc;
        if (ts[i]->rows != grad->rows || ts[i]->cols != grad->cols)
            return fail(CODA_E_DIMENSION, "%s has shape (%lld,%lld), expected (%lld,%lld)", nm[i],
                        (long long)ts[i]->rows, (long long)ts[i]->cols, (long long)grad->rows,
                        (long long)grad->cols);
    }
    if (h <= 0 || h % 32 || 2 * h > grad->cols)
        return fail(CODA_E_DIMENSION, "compact RoPE width h=%lld must be a positive multiple of 32 with 2h <= n",
                    (long long)h);
    const coda_tensor_t* tb[2] = {cos_c, sin_c};
    for (int i = 0; i < 2; ++i) {
        if ((rc = check_tensor2d(tb[i], i ? "sin_c" : "cos_c", CODA_BF16))) return rc;
        if (tb[i]->rows != grad->rows || tb[i]->cols != h / 2)
            return fail(CODA_E_DIMENSION, "compact table must be (%lld, %lld)", (long long)grad->rows,
                        (long long)(h / 2));
    }
    DeviceGuard dg;
    if ((rc = bind_device(grad->ptr, dg))) return rc;
    // deep-load variant when rows split into whole 6 (or 3) x 2048-column sweeps (16-B aligned rows)
    int U = grad->cols % (6 * 2048) == 0 ? 6 : 3;
    bool deep = true;
#ifdef CODA_EXPERIMENTS
    if (opts().rope_u == 1) deep = false;
    else if (opts().rope_u == 3 || opts().rope_u == 6) U = opts().rope_u;
#endif
    deep = deep && grad->cols % (U * 2048) == 0 && grad->ld % 8 == 0 && rotated->ld % 8 == 0 &&
           grad_z->ld % 8 == 0 && cos_c->ld % 4 == 0 && sin_c->ld % 4 == 0;
    if (deep) {
        const int64_t items = grad->rows * (grad->cols / (U * 2048));
        const unsigned g = (unsigned)std::min<int64_t>(items, (int64_t)num_sms() * 8);
        auto kern = U == 6 ? coda::coda_rope_backward_stat_deep_kernel<6> : coda::coda_rope_backward_stat_deep_kernel<3>;
        return launch_pdl(kern, dim3(g), dim3(256), 0, (cudaStream_t)stream, 1,
                          "coda::coda_rope_backward_stat_deep_kernel",
                          (const __nv_bfloat16*)grad->ptr, grad->ld, (const __nv_bfloat16*)rotated->ptr, rotated->ld,
                          (const __nv_bfloat16*)cos_c->ptr, cos_c->ld, (const __nv_bfloat16*)sin_c->ptr, sin_c->ld, h,
                          grad->rows, grad->cols, (__nv_bfloat16*)grad_z->ptr, grad_z->ld, rowdot, ld_rowdot);
    }
    const unsigned grid = (unsigned)(grad->rows < 148 * 8 ? grad->rows : 148 * 8);
    return launch_pdl(coda::coda_rope_backward_stat128_compact_kernel, dim3(grid), dim3(256), 0,
                      (cudaStream_t)stream, 1, "coda::coda_rope_backward_stat128_compact_kernel",
                      (const __nv_bfloat16*)grad->ptr, grad->ld, (const __nv_bfloat16*)rotated->ptr, rotated->ld,
                      (const __nv_bfloat16*)cos_c->ptr, cos_c->ld, (const __nv_bfloat16*)sin_c->ptr, sin_c->ld, h,
                      grad->rows, grad->cols, (__nv_bfloat16*)grad_z->ptr, grad_z->ld, rowdot, ld_rowdot);
}

int coda_rope_backward_stat(const coda_tensor_t* grad, const coda_tensor_t* rotated, const coda_tensor_t* cos,
                            const coda_tensor_t* sin, const int32_t* block_start, int64_t nb, coda_tensor_t* grad_z,
                            float* rowdot, int64_t ld_rowdot, void* stream) {
    if (!grad) return fail(CODA_E_BINDING, "null grad");
    const int dt = grad->dtype;
    if (dt != CODA_BF16 && dt != CODA_F32) return fail(CODA_E_CONFIG, "rope_backward_stat: bad dtype");
    int rc;
    const coda_tensor_t* ts[5] = {grad, rotated, cos, sin, grad_z};
    const char* nm[5] = {"grad", "rotated", "cos", "sin", "grad_z"};
    for (int i = 0; i < 5; ++i) {
        if ((rc = check_tensor2d(ts[i], nm[i], dt))) return rc;
        if (ts[i]->rows != grad->rows || ts[i]->cols != grad->cols)
            return fail(CODA_E_DIMENSION, "%s has shape (%lld,%lld), expected (%lld,%lld)", nm[i],
                        (long long)ts[i]->rows, (long long)ts[i]->cols, (long long)grad->rows,
                        (long long)grad->cols);
    }
    if (grad->cols % 2) return fail(CODA_E_DIMENSION, "rotary width must be even, got %lld", (long long)grad->cols);
    DeviceGuard dg;
    if ((rc = bind_device(grad->ptr, dg))) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (block_start == nullptr) {
        if (nb != (grad->cols + 127) / 128) return fail(CODA_E_DIMENSION, "rope_backward_stat: nb != ceil(n/128)");
        const unsigned grid = (unsigned)(grad->rows < 148 * 8 ? grad->rows : 148 * 8);
        if (dt == CODA_BF16) {
            return launch_pdl(coda::coda_rope_backward_stat128_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, st, 1, "coda::coda_rope_backward_stat128_kernel<__nv_bfloat16>",
        (const __nv_bfloat16*)grad->ptr, grad->ld, (const __nv_bfloat16*)rotated->ptr, rotated->ld,
                (const __nv_bfloat16*)cos->ptr, cos->ld, (const __nv_bfloat16*)sin->ptr, sin->ld, grad->rows,
                grad->cols, (__nv_bfloat16*)grad_z->ptr, grad_z->ld, rowdot, ld_rowdot);
        } else {
            return launch_pdl(coda::coda_rope_backward_stat128_kernel<float>, dim3(grid), dim3(256), 0, st, 1, "coda::coda_rope_backward_stat128_kernel<float>",
        (const float*)grad->ptr, grad->ld, (const float*)rotated->ptr, rotated->ld, (const float*)cos->ptr,
                cos->ld, (const float*)sin->ptr, sin->ld, grad->rows, grad->cols, (float*)grad_z->ptr, grad_z->ld,
                rowdot, ld_rowdot);
        }
        return cuda_check(cudaGetLastError(), "rope_backward_stat128");
    }
    const size_t smem = (size_t)grad->cols * 4;
    if (smem > 200 * 1024) return fail(CODA_E_CONFIG, "rope_backward_stat: row too wide (%lld)", (long long)grad->cols);
    if (dt == CODA_BF16) {
        auto k = coda::coda_rope_backward_stat_kernel<__nv_bfloat16>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        return launch_pdl(k, dim3((unsigned)grad->rows), dim3(256), smem, st, 1, "k",
        (const __nv_bfloat16*)grad->ptr, grad->ld, (const __nv_bfloat16*)rotated->ptr, rotated->ld,
            (const __nv_bfloat16*)cos->ptr, cos->ld, (const __nv_bfloat16*)sin->ptr, sin->ld, grad->cols, block_start,
            nb, (__nv_bfloat16*)grad_z->ptr, grad_z->ld, rowdot, ld_rowdot);
    } else {
        auto k = coda::coda_rope_backward_stat_kernel<float>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        return launch_pdl(k, dim3((unsigned)grad->rows), dim3(256), smem, st, 1, "k",
        (const float*)grad->ptr, grad->ld, (const float*)rotated->ptr, rotated->ld, (const float*)cos->ptr, cos->ld,
            (const float*)sin->ptr, sin->ld, grad->cols, block_start, nb, (float*)grad_z->ptr, grad_z->ld, rowdot,
            ld_rowdot);
    }
    return cuda_check(cudaGetLastError(), "rope_backward_stat");
}

int coda_combine_row_pieces(const float* pieces, int64_t m, int64_t np, int64_t ldp, const int32_t* block_ptr,
                            int64_t nb, int pairs, float* out, int64_t ldo, void* stream) {
    if (m <= 0 || np <= 0 || nb <= 0) return fail(CODA_E_DIMENSION, "combine_row_pieces: empty");
    int rc;
    DeviceGuard dg;
    if ((rc = bind_device(pieces, dg))) return rc;
    return launch_pdl(coda::coda_combine_row_pieces_kernel, dim3(grid1d(m * nb, 256)), dim3(256), 0, (cudaStream_t)stream, 1, "coda::coda_combine_row_pieces_kernel",
        pieces, m, np, ldp, block_ptr, nb, pairs, out, ldo);
}

int coda_combine_col_pieces(const float* pieces, int64_t np, int64_t n, int64_t ldp, const int32_t* block_ptr,
                            int64_t nb, float* out, int64_t ldo, void* stream) {
    if (n <= 0 || np <= 0 || nb <= 0) return fail(CODA_E_DIMENSION, "combine_col_pieces: empty");
    if (nb > 65535) return fail(CODA_E_CONFIG, "combine_col_pieces: too many blocks");
    int rc;
    DeviceGuard dg;
    if ((rc = bind_device(pieces, dg))) return rc;
    dim3 grid(grid1d(n, 256), (unsigned)nb);
    return launch_pdl(coda::coda_combine_col_pieces_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, 1, "coda::coda_combine_col_pieces_kernel",
        pieces, np, n, ldp, block_ptr, nb, out, ldo);
}

int coda_split_operand(const coda_tensor_t* src, int k_axis, int64_t kp, const int32_t pattern[6],
                       coda_tensor_t* dst, void* stream) {
    int rc;
    if ((rc = check_tensor2d(src, "split src", CODA_F32))) return rc;
    if ((rc = check_tensor2d(dst, "split dst", CODA_BF16))) return rc;
    const int64_t kk = k_axis ? src->cols : src->rows;
    if (kp < kk) return fail(CODA_E_DIMENSION, "split: kp < K");
    const int64_t drows = k_axis ? src->rows : 6 * kp, dcols = k_axis ? 6 * kp : src->cols;
    if (dst->rows != drows || dst->cols != dcols) return fail(CODA_E_DIMENSION, "split: dst shape mismatch");
    coda::SplitPattern pat;
    for (int i = 0; i < 6; ++i) {
        if (pattern[i] < 0 || pattern[i] > 2) return fail(CODA_E_CONFIG, "split: bad pattern");
        pat.t[i] = pattern[i];
    }
    DeviceGuard dg;
    if ((rc = bind_device(src->ptr, dg))) return rc;
    return launch_pdl(coda::coda_split_operand_kernel, dim3(grid1d(drows * dcols, 256)), dim3(256), 0, (cudaStream_t)stream, 1, "coda::coda_split_operand_kernel",
        (const float*)src->ptr, src->rows, src->cols, src->ld, k_axis, kp, pat, (__nv_bfloat16*)dst->ptr, drows,
        dcols, dst->ld);
}

int coda_scale_rows(const coda_tensor_t* src, const float* scale, coda_tensor_t* dst, void* stream) {
    int rc;
    if ((rc = check_tensor2d(src, "scale_rows src", CODA_BF16))) return rc;
    if ((rc = check_tensor2d(dst, "scale_rows dst", CODA_BF16))) return rc;
    if (!scale) return fail(CODA_E_BINDING, "scale_rows: null scale vector");
    if (src->rows != dst->rows || src->cols != dst->cols) return fail(CODA_E_DIMENSION, "scale_rows: shapes differ");
    DeviceGuard dg;
    if ((rc = bind_device(src->ptr, dg))) return rc;
    const int vec = src->cols % 8 == 0 && src->ld % 8 == 0 && dst->ld % 8 == 0;
    const int64_t work = vec ? src->rows * (src->cols / 8) : src->rows * src->cols;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 8));
    return launch_pdl(coda::coda_scale_rows_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, 1,
                      "coda::coda_scale_rows_kernel", (const __nv_bfloat16*)src->ptr, src->rows, src->cols, src->ld,
                      scale, (__nv_bfloat16*)dst->ptr, dst->ld, vec);
}

int coda_convert_f32_bf16(const coda_tensor_t* src, coda_tensor_t* dst, void* stream) {
    if (!src || !dst || !src->ptr || !dst->ptr) return fail(CODA_E_BINDING, "convert: null tensor");
    if (src->dtype != CODA_F32 || dst->dtype != CODA_BF16) return fail(CODA_E_BINDING, "convert: dtypes");
    if (src->rows != dst->rows || src->cols != dst->cols) return fail(CODA_E_DIMENSION, "convert: shapes differ");
    int rc;
    DeviceGuard dg;
    if ((rc = bind_device(src->ptr, dg))) return rc;
    const int vec = src->ld % 4 == 0 && dst->ld % 8 == 0 && reinterpret_cast<uintptr_t>(src->ptr) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(dst->ptr) % 16 == 0;
    const int64_t work = vec ? src->rows * (src->cols / 8) : src->rows;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 8));
    return launch_pdl(coda::coda_convert_f32_bf16_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, 1,
                      "coda::coda_convert_f32_bf16_kernel", (const float*)src->ptr, src->rows, src->cols, src->ld,
                      (__nv_bfloat16*)dst->ptr, dst->ld, vec);
}

}  // extern "C"
