// fvb.cu -- libfvb.so: the C ABI declared in include/fvb.h (step, plans,
// graphs, errors).  Kernels live in the other translation units (host.h).
//
// Build (build.py): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
// --fmad=false -- no FMA contraction, for bit parity with the numpy/Python
// reference.

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "fused2d.cuh"
#include "fused2d_tma.cuh"
#include "fused3d.cuh"
#include "fused3d_warp.cuh"  // the one-warp kernel's shared memory (fvb_fused_smem_bytes)
#include "host.h"

using namespace fvb;

// ---------------------------------------------------------------------------
// errors and device facts
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;

namespace fvb {

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(FVB_ECUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
    return FVB_OK;
}

long long ipow_h(long long b, int e) {
    long long r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

int validate_shape(int dim, int p, int64_t T) {
    if (dim != 2 && dim != 3) return fail(FVB_EINVAL, "dim must be 2 or 3, got %d", dim);
    if (p < 2) return fail(FVB_EINVAL, "patch_size must be >= 2, got %d", p);
    if (T < 1) return fail(FVB_EINVAL, "patch_count must be >= 1, got %lld", (long long)T);
    if (ipow_h(p + 2, dim) > (1LL << 30)) return fail(FVB_EINVAL, "patch too large (p=%d)", p);
    return FVB_OK;
}

int sm_count() {
    static PerDevice n_dev;
    int& n = n_dev();
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

int smem_optin() {
    static PerDevice n_dev;
    int& n = n_dev();
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (n <= 0) n = 227 * 1024;
    }
    return n;
}

// 4-D fp64 tiled tensor map (TMA) over a batch array; the driver's encoder
// is looked up once through the runtime (no libcuda link).  False if the
// driver lacks it or rejects the description.
bool tensor_map_4d(CUtensorMap* tm, const void* base, const unsigned long long dims[4],
                   const unsigned long long strides_bytes[3], const unsigned box[4]) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (encode == nullptr) return false;
    cuuint64_t d[4], st[3];
    cuuint32_t b[4], e[4] = {1, 1, 1, 1};
    for (int i = 0; i < 4; ++i) d[i] = dims[i], b[i] = box[i];
    for (int i = 0; i < 3; ++i) st[i] = strides_bytes[i];
    return encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), d, st, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

long long blocks_for(long long work, int threads, int per_sm) {
    long long b = (work + threads - 1) / threads;
    long long cap = (long long)sm_count() * per_sm;
    if (b > cap) b = cap;
    return b < 1 ? 1 : b;
}

// Launch tuning: initialised from the environment, changed by fvb_set_tuning.
static int g_tuning[3];
static std::once_flag g_tuning_once;
static void tuning_init() {
    const char* names[3] = {"FVB_TUNE_PENCIL_VARIANT", "FVB_TUNE_SLAB_VARIANT", "FVB_TUNE_REDUCE_FILTER"};
    const int defaults[3] = {0, 0, -1};
    for (int i = 0; i < 3; ++i) {
        const char* e = getenv(names[i]);
        g_tuning[i] = e ? atoi(e) : defaults[i];
    }
}

int tuning(int key) {
    std::call_once(g_tuning_once, tuning_init);
    return (key >= 0 && key < 3) ? g_tuning[key] : 0;
}

// Physics policy selection (fvb_set_physics): from FVB_PHYSICS, default Euler.
static std::atomic<int> g_physics{-1};
int physics() {
    int v = g_physics.load();
    if (v < 0) {
        const char* e = getenv("FVB_PHYSICS");
        v = (e && atoi(e) == FVB_PHYSICS_EULER_PLAIN) ? FVB_PHYSICS_EULER_PLAIN : FVB_PHYSICS_EULER;
        int expect = -1;
        g_physics.compare_exchange_strong(expect, v);
        v = g_physics.load();
    }
    return v;
}

}  // namespace fvb

extern "C" int fvb_set_tuning(int key, int value) {
    if (key < 0 || key >= 3) return fail(FVB_EINVAL, "unknown tuning key %d", key);
    std::call_once(g_tuning_once, tuning_init);
    g_tuning[key] = value;
    return FVB_OK;
}

extern "C" int fvb_get_tuning(int key, int* value) {
    if (key < 0 || key >= 3) return fail(FVB_EINVAL, "unknown tuning key %d", key);
    *value = tuning(key);
    return FVB_OK;
}

extern "C" int fvb_set_physics(int id) {
    if (id != FVB_PHYSICS_EULER && id != FVB_PHYSICS_EULER_PLAIN) return fail(FVB_EINVAL, "unknown physics %d", id);
    g_physics.store(id);
    return FVB_OK;
}

extern "C" int fvb_get_physics(int* id) {
    if (id == nullptr) return fail(FVB_EINVAL, "null argument");
    *id = physics();
    return FVB_OK;
}

extern "C" const char* fvb_version(void) { return "fvb 0.1.0 sm_100a"; }
extern "C" const char* fvb_last_error(void) { return g_last_error.c_str(); }

static int validate_run(double dt, double h, double gamma) {
    if (!(dt > 0.0)) return fail(FVB_EINVAL, "dt must be positive, got %g", dt);
    if (!(h > 0.0)) return fail(FVB_EINVAL, "h must be positive, got %g", h);
    if (!(gamma > 1.0)) return fail(FVB_EINVAL, "adiabatic exponent must exceed 1, got %g", gamma);
    return FVB_OK;
}

// ---------------------------------------------------------------------------
// fused flavour: pencil kernel for 2D p in FVB_PENCIL_SIZES, else generic
// ---------------------------------------------------------------------------
static bool uses_pencil(int dim, int p) {
    if (dim != 2) return false;
    switch (p) {
#define FVB_CASE(P) case P:
        FVB_PENCIL_SIZES(FVB_CASE)
#undef FVB_CASE
        return true;
        default:
            return false;
    }
}

static bool uses_slab(int dim, int p) {
    if (dim != 3) return false;
    switch (p) {
#define FVB_CASE(P) case P:
        FVB_SLAB_SIZES(FVB_CASE)
#undef FVB_CASE
        return true;
        default:
            return false;
    }
}

// shared memory of the default 2D pencil launch (pencil.cu: one warp; p | 32:
// the TMA-streamed ring of 3 two-row slots, else the 3-row cp.async ring)
template <int P>
static constexpr int64_t pencil_default_smem() {
    if constexpr (32 % P == 0) {
        return (int64_t)pencil_tma_smem<P, 3, 2, 4>();
    } else {
        return (int64_t)pencil_smem_per_warp<P, 1, 3, 4>();
    }
}
static int64_t pencil_smem_bytes(int p) {
    switch (p) {
#define FVB_CASE(P) \
    case P:         \
        return pencil_default_smem<P>();
        FVB_PENCIL_SIZES(FVB_CASE)
#undef FVB_CASE
    }
    return 0;
}

// shared memory of the default 3D launch (slab3d.cu): p = 8 one warp per
// patch with a 2-plane ring, other p one two-warp slot with a 4-plane ring
static int64_t slab_smem_bytes(int p) {
    switch (p) {
#define FVB_CASE(P) \
    case P:         \
        return (int64_t)(P == 8 ? sizeof(slabw::WarpSmem<P, 2, 5>)                                \
                                : (slab::Geo3<P>::TH < 32 ? 32 / slab::Geo3<P>::TH : 1) *          \
                                      slab_smem_per_slot<P, 4, 5>());
        FVB_SLAB_SIZES(FVB_CASE)
#undef FVB_CASE
    }
    return 0;
}

static int launch_fused(int dim, const StepArgs& a, bool reduce, cudaStream_t st) {
    if (uses_slab(dim, a.p)) {
        switch (a.p) {
#define FVB_CASE(P) \
    case P:         \
        return slab_launch<P>(a, reduce, st);
            FVB_SLAB_SIZES(FVB_CASE)
#undef FVB_CASE
        }
    }
    if (uses_pencil(dim, a.p)) {
        switch (a.p) {
#define FVB_CASE(P) \
    case P:         \
        return pencil_launch<P>(a, reduce, st);
            FVB_PENCIL_SIZES(FVB_CASE)
#undef FVB_CASE
        }
    }
    return launch_generic(dim, a, reduce, st);
}

static int fused_fits(int dim, int p) {
    if (!uses_pencil(dim, p) && !uses_slab(dim, p) && generic_smem_bytes(dim, p) > smem_optin())
        return fail(FVB_ELIMIT,
                    "(p+2)^d staging for d=%d p=%d needs %lld B shared memory > %d B per CTA; "
                    "use the cascade or graph flavour",
                    dim, p, generic_smem_bytes(dim, p), smem_optin());
    return FVB_OK;
}

extern "C" int fvb_fused_limit(int dim, int* max_p) {
    if (dim != 2 && dim != 3) return fail(FVB_EINVAL, "dim must be 2 or 3, got %d", dim);
    int p = 2;
    while (generic_smem_bytes(dim, p + 1) <= smem_optin() || uses_pencil(dim, p + 1) ||
           uses_slab(dim, p + 1))
        ++p;
    *max_p = p;
    return FVB_OK;
}

extern "C" int fvb_fused_smem_bytes(int dim, int p, int64_t* bytes) {
    int rc = validate_shape(dim, p, 1);
    if (rc) return rc;
    *bytes = uses_pencil(dim, p) ? pencil_smem_bytes(p)
             : uses_slab(dim, p)  ? slab_smem_bytes(p)
                                  : generic_smem_bytes(dim, p);
    return FVB_OK;
}

// ---------------------------------------------------------------------------
// plans: scratch arena (cascade / graph) and the task graph
// ---------------------------------------------------------------------------
struct fvb_plan {
    int flavour, dim, p, chunks;
    int physics = FVB_PHYSICS_EULER;  // policy selected at creation (fvb_set_physics)
    int layout = kLayoutSoA;
    long long T;
    double* scratch = nullptr;  // flux + lambda temporaries (cascade / graph), owned
    size_t scratch_bytes = 0;
    bool external_scratch = false;  // temporaries supplied by the caller (fvb_plan_create_ext)
    std::mutex mu;                  // held by step_any while a cached plan runs
    CascadeArgs ca{};
    // graph flavour: one instantiated graph per (with_reduction, has_lam_patch)
    cudaGraphExec_t exec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    cudaGraph_t graph[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // kept: exec node updates need its node handles
    int64_t graph_nodes[2][2] = {{0, 0}, {0, 0}};
    std::vector<cudaGraphNode_t> kernel_nodes[2][2];
    std::vector<int> node_chunk[2][2];  // chunk of each kernel node
    std::vector<int> node_kind[2][2];   // 0 copy, 1 flux, 2 lambda, 3 acc, 4 reduce
    std::vector<int> node_axis[2][2];
    StepArgs bound[2][2]{};
};

static void chunk_range(long long T, int chunks, int c, long long* t0, long long* t1) {
    const long long base = T / chunks, rem = T % chunks;
    *t0 = c * base + (c < rem ? c : rem);
    *t1 = *t0 + base + (c < rem ? 1 : 0);
}

static int alloc_scratch(fvb_plan* pl) {
    const int n = pl->dim + 2;
    const long long R = (pl->p + 2) * ipow_h(pl->p, pl->dim - 1);
    const size_t per_axis = (size_t)(n + 1) * (size_t)pl->T * (size_t)R;
    pl->scratch_bytes = per_axis * pl->dim * sizeof(double);
    FVB_CUDA(cudaMalloc(&pl->scratch, pl->scratch_bytes));
    for (int a = 0; a < pl->dim; ++a) {
        pl->ca.tmp_flux[a] = pl->scratch + a * per_axis;
        pl->ca.tmp_lam[a] = pl->scratch + a * per_axis + (size_t)n * pl->T * R;
    }
    for (int a = pl->dim; a < 3; ++a) pl->ca.tmp_flux[a] = pl->ca.tmp_lam[a] = nullptr;
    return FVB_OK;
}

// Build the task-graph flavour: per chunk c the lifted per-patch DAG
// (kernelgraph.py:215-247): copy, flux_n, lambda_n are roots; acc_n waits for
// copy, flux_n, lambda_n and acc_{n-1}; reduce waits for acc_{d-1}.  Chunks
// share no edges (no cross-patch dependencies, test_kernelgraph.py:105-108);
// the zeroing of the eigenvalue outputs is one memset root before every reduce.
static int build_graph(fvb_plan* pl, const StepArgs& a, bool reduce, bool has_lp) {
    const int ri = reduce ? 1 : 0, li = has_lp ? 1 : 0;
    cudaGraph_t g;
    FVB_CUDA(cudaGraphCreate(&g, 0));
    const int d = pl->dim;
    const CascadeFns fns = cascade_fns(d, pl->physics);
    std::vector<cudaGraphNode_t> memset_nodes;
    if (reduce) {
        cudaMemsetParams mp{};
        mp.dst = a.lam_bits;
        mp.value = 0;
        mp.elementSize = 4;
        mp.width = 2;
        mp.height = 1;
        mp.pitch = 0;
        cudaGraphNode_t n;
        FVB_CUDA(cudaGraphAddMemsetNode(&n, g, nullptr, 0, &mp));
        memset_nodes.push_back(n);
        if (has_lp) {
            mp.dst = a.lam_patch;
            mp.width = (size_t)(2 * pl->T);
            FVB_CUDA(cudaGraphAddMemsetNode(&n, g, nullptr, 0, &mp));
            memset_nodes.push_back(n);
        }
    }
    auto& kn = pl->kernel_nodes[ri][li];
    auto& kchunk = pl->node_chunk[ri][li];
    auto& kkind = pl->node_kind[ri][li];
    auto& kaxis = pl->node_axis[ri][li];
    kn.clear(), kchunk.clear(), kkind.clear(), kaxis.clear();
    int64_t nodes = (int64_t)memset_nodes.size();
    const long long Mi = ipow_h(a.p, d), R = (a.p + 2) * ipow_h(a.p, d - 1);
    for (int c = 0; c < pl->chunks; ++c) {
        StepArgs sa = a;
        chunk_range(pl->T, pl->chunks, c, &sa.t0, &sa.t1);
        if (sa.t1 <= sa.t0) continue;
        CascadeArgs ca = pl->ca;
        ca.s = sa;
        const long long span = sa.t1 - sa.t0;
        const unsigned gi = (unsigned)blocks_for(span * Mi, kEltThreads, 16);
        const unsigned gr = (unsigned)blocks_for(span * R, kEltThreads, 16);
        auto add = [&](void* fn, unsigned grid, unsigned block, void** args,
                       const std::vector<cudaGraphNode_t>& deps, int kind, int axis,
                       cudaGraphNode_t* out) -> int {
            cudaKernelNodeParams kp{};
            kp.func = fn;
            kp.gridDim = dim3(grid);
            kp.blockDim = dim3(block);
            kp.sharedMemBytes = 0;
            kp.kernelParams = args;
            FVB_CUDA(cudaGraphAddKernelNode(out, g, deps.data(), deps.size(), &kp));
            kn.push_back(*out), kchunk.push_back(c), kkind.push_back(kind), kaxis.push_back(axis);
            ++nodes;
            return FVB_OK;
        };
        cudaGraphNode_t copy_n, flux_n[3], lam_n[3], acc_n[3], red_n;
        void* a_args[] = {&sa};
        int rc = add(fns.copy, gi, kEltThreads, a_args, {}, 0, -1, &copy_n);
        if (rc) return rc;
        int axes[3] = {0, 1, 2};
        for (int ax = 0; ax < d; ++ax) {
            void* f_args[] = {&ca, &axes[ax]};
            if ((rc = add(fns.flux, gr, kEltThreads, f_args, {}, 1, ax, &flux_n[ax]))) return rc;
        }
        for (int ax = 0; ax < d; ++ax) {
            void* f_args[] = {&ca, &axes[ax]};
            if ((rc = add(fns.lam, gr, kEltThreads, f_args, {}, 2, ax, &lam_n[ax]))) return rc;
        }
        for (int ax = 0; ax < d; ++ax) {
            std::vector<cudaGraphNode_t> deps = {copy_n, flux_n[ax], lam_n[ax]};
            if (ax > 0) deps.push_back(acc_n[ax - 1]);
            void* f_args[] = {&ca, &axes[ax]};
            if ((rc = add(fns.acc, gi, kEltThreads, f_args, deps, 3, ax, &acc_n[ax]))) return rc;
        }
        if (reduce) {
            std::vector<cudaGraphNode_t> deps = memset_nodes;
            deps.push_back(acc_n[d - 1]);
            if ((rc = add(fns.reduce, gi, kReduceThreads, a_args, deps, 4, -1, &red_n))) return rc;
        }
    }
    cudaGraphExec_t ex;
    FVB_CUDA(cudaGraphInstantiate(&ex, g, 0));
    pl->graph[ri][li] = g;
    pl->exec[ri][li] = ex;
    pl->graph_nodes[ri][li] = nodes;
    pl->bound[ri][li] = a;
    return FVB_OK;
}

// Re-point an instantiated graph at new buffers / run parameters.
static int rebind_graph(fvb_plan* pl, const StepArgs& a, bool reduce, bool has_lp) {
    const int ri = reduce ? 1 : 0, li = has_lp ? 1 : 0;
    const StepArgs& b = pl->bound[ri][li];
    if (b.q_in == a.q_in && b.q_out == a.q_out && b.scale == a.scale && b.gamma == a.gamma &&
        b.lam_bits == a.lam_bits && b.lam_patch == a.lam_patch && b.layout == a.layout &&
        b.dt_dev == a.dt_dev && b.dt_patch == a.dt_patch && b.h == a.h && b.in_tab == a.in_tab &&
        b.out_tab == a.out_tab)
        return FVB_OK;
    // memset destinations changed -> rebuild; kernel args -> in-place update
    if (b.lam_bits != a.lam_bits || b.lam_patch != a.lam_patch) {
        cudaGraphExecDestroy(pl->exec[ri][li]);
        cudaGraphDestroy(pl->graph[ri][li]);
        pl->graph[ri][li] = nullptr;
        pl->exec[ri][li] = nullptr;
        return build_graph(pl, a, reduce, has_lp);
    }
    const CascadeFns fns = cascade_fns(pl->dim, pl->physics);
    auto& kn = pl->kernel_nodes[ri][li];
    const long long Mi = ipow_h(a.p, pl->dim), R = (a.p + 2) * ipow_h(a.p, pl->dim - 1);
    for (size_t i = 0; i < kn.size(); ++i) {
        StepArgs sa = a;
        chunk_range(pl->T, pl->chunks, pl->node_chunk[ri][li][i], &sa.t0, &sa.t1);
        CascadeArgs ca = pl->ca;
        ca.s = sa;
        int axis = pl->node_axis[ri][li][i];
        const int kind = pl->node_kind[ri][li][i];
        const long long span = sa.t1 - sa.t0;
        cudaKernelNodeParams kp{};
        void* a_args[] = {&sa};
        void* f_args[] = {&ca, &axis};
        switch (kind) {
            case 0: kp.func = fns.copy; break;
            case 1: kp.func = fns.flux; break;
            case 2: kp.func = fns.lam; break;
            case 3: kp.func = fns.acc; break;
            default: kp.func = fns.reduce; break;
        }
        const bool interior = (kind == 0 || kind == 3 || kind == 4);
        kp.gridDim = dim3((unsigned)blocks_for(span * (interior ? Mi : R), kEltThreads, 16));
        kp.blockDim = dim3(kind == 4 ? kReduceThreads : kEltThreads);
        kp.kernelParams = (kind == 0 || kind == 4) ? a_args : f_args;
        FVB_CUDA(cudaGraphExecKernelNodeSetParams(pl->exec[ri][li], kn[i], &kp));
        FVB_CUDA(cudaGraphKernelNodeSetParams(kn[i], &kp));  // the graph too: a capture embeds a copy of it
    }
    pl->bound[ri][li] = a;
    return FVB_OK;
}

// Per-call options of plan_run beyond the uniform step.
struct RunOpts {
    const double* dt_dev = nullptr;    // dt read on the device (fvb_step_dt)
    const double* dt_patch = nullptr;  // per-patch dt (fvb_step_lts)
    const double* const* in_tab = nullptr;  // SHARED mode pointer tables (fvb_step_table)
    double* const* out_tab = nullptr;
    long long t0 = 0, t1 = -1;  // patch range of the batch (fvb_step_range); t1 < 0: all
    bool zero = true;           // zero lam (and lam_patch over the range) first
};

// Reduction slots of the fused flavour (common.cuh reduce_epilogue), one per
// (device, stream): launches on one stream are ordered, so they share it.
// cudaStreamPerThread is one handle for many streams: its slots are keyed by
// the host thread too (stream_thread_key).  (A stream destroyed with work pending whose handle
// is reused for a new stream would share the slot with that work: destroy
// streams after synchronising them.)  Made and zeroed on first use; a
// launch being captured into a graph uses none and zeroes the output with a
// memset node instead.
static std::mutex g_slot_mu;
static std::map<std::tuple<int, void*, size_t>, RedSlot*> g_slots;

static RedSlot* reduction_slot(cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    // a captured launch gets no slot: the graph may be replayed on any stream,
    // concurrently with launches on the capturing one
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return nullptr;
    }
    const auto key = std::make_tuple(dev, (void*)st, stream_thread_key(st));
    std::lock_guard<std::mutex> lk(g_slot_mu);
    auto it = g_slots.find(key);
    if (it != g_slots.end()) return it->second;
    RedSlot* s = nullptr;
    if (cudaMalloc(&s, sizeof(RedSlot)) != cudaSuccess || cudaMemset(s, 0, sizeof(RedSlot)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        cudaGetLastError();
        if (s) cudaFree(s);
        return nullptr;
    }
    g_slots[key] = s;
    return s;
}

// dt_dev != null: dt is read on the device (fvb_step_dt); dt_patch != null:
// every patch has its own dt (fvb_step_lts).  Either way `dt` is ignored.
static int plan_run(fvb_plan* pl, const double* q_in, double* q_out, double dt, double h,
                    double gamma, int with_reduction, double* lam, double* lam_patch,
                    cudaStream_t st, const RunOpts& o = RunOpts()) {
    const RelaxedCapture relaxed;  // a task graph instantiated eagerly inside a user's capture
    const double* dt_dev = o.dt_dev;
    const double* dt_patch = o.dt_patch;
    int rc = validate_run((dt_dev != nullptr || dt_patch != nullptr) ? 1.0 : dt, h, gamma);
    if (rc) return rc;
    const bool tables = o.in_tab != nullptr || o.out_tab != nullptr;
    if (tables && (o.in_tab == nullptr || o.out_tab == nullptr))
        return fail(FVB_EINVAL, "pointer tables come in pairs (input and output)");
    if (!tables && (q_in == nullptr || q_out == nullptr)) return fail(FVB_EINVAL, "null batch pointer");
    const long long t0 = o.t0, t1 = o.t1 < 0 ? pl->T : o.t1;
    if (t0 < 0 || t1 > pl->T || t0 >= t1) return fail(FVB_EINVAL, "patch range [%lld, %lld) outside [0, %lld)",
                                                      t0, t1, pl->T);
    const bool reduce = with_reduction != 0;
    if (reduce && lam == nullptr) return fail(FVB_EINVAL, "with_reduction needs lam_dev");
    StepArgs a{};
    a.q_in = q_in;
    a.q_out = q_out;
    a.T = pl->T;
    a.t0 = t0;
    a.t1 = t1;
    a.scale = dt / h;
    a.gamma = gamma;
    a.lam_bits = reduce ? reinterpret_cast<unsigned long long*>(lam) : nullptr;
    a.lam_patch = reduce ? lam_patch : nullptr;
    a.p = pl->p;
    a.layout = tables ? kLayoutAoS : pl->layout;  // per-patch arrays are AoS (memory.py:60-64)
    a.in = layout_strides(a.layout, pl->T, ipow_h(pl->p + 2, pl->dim), pl->dim + 2);
    a.out = layout_strides(a.layout, pl->T, ipow_h(pl->p, pl->dim), pl->dim + 2);
    a.in_tab = o.in_tab;
    a.out_tab = o.out_tab;
    // folded faces need an exact 0.5*dt/h, the fast paths a sane gamma (fused2d.cuh)
    a.fast = (a.scale >= 0x1p-1000 && a.scale <= 0x1p+1000 && gamma <= 0x1p+100) ? 1 : 0;
    a.dt_dev = dt_dev;  // the kernels then form dt/h and the same range check on the device
    a.dt_patch = dt_patch;
    a.h = h;
    a.physics = pl->physics;
    if (dt_dev != nullptr || dt_patch != nullptr) a.scale = 0.0, a.fast = 0;
    const bool has_lp = a.lam_patch != nullptr;
    if (pl->flavour == FVB_GRAPH) {
        if (t0 != 0 || t1 != pl->T || !o.zero)
            return fail(FVB_EINVAL, "the task graph runs whole batches (no patch range)");
        const int ri = reduce ? 1 : 0, li = has_lp ? 1 : 0;
        if (pl->exec[ri][li] == nullptr) {
            if ((rc = build_graph(pl, a, reduce, has_lp))) return rc;
        } else if ((rc = rebind_graph(pl, a, reduce, has_lp))) {
            return rc;
        }
        // inside a user's stream capture the task graph goes in as a child
        // graph node (a graph launch cannot be captured)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaGraph_t cap = nullptr;
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        FVB_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cap, &deps, &ndeps));
        if (cs == cudaStreamCaptureStatusActive) {
            cudaGraphNode_t child;
            FVB_CUDA(cudaGraphAddChildGraphNode(&child, cap, deps, ndeps, pl->graph[ri][li]));
            FVB_CUDA(cudaStreamUpdateCaptureDependencies(st, &child, 1, cudaStreamSetCaptureDependencies));
            return FVB_OK;
        }
        FVB_CUDA(cudaGraphLaunch(pl->exec[ri][li], st));
        return FVB_OK;
    }
    if (pl->flavour == FVB_FUSED) {
        // fused kernels write every patch's lam_patch entry and, through the
        // slot, the result itself: no memset launch before the kernel
        if (reduce) {
            a.red_slot = reduction_slot(st);
            a.lam_accumulate = o.zero ? 0 : 1;
            if (a.red_slot == nullptr && o.zero) FVB_CUDA(cudaMemsetAsync(lam, 0, sizeof(double), st));
        }
        return launch_fused(pl->dim, a, reduce, st);
    }
    if (reduce && o.zero) {
        FVB_CUDA(cudaMemsetAsync(lam, 0, sizeof(double), st));
        if (has_lp) FVB_CUDA(cudaMemsetAsync(lam_patch + t0, 0, sizeof(double) * (t1 - t0), st));
    }
    CascadeArgs ca = pl->ca;
    ca.s = a;
    return launch_cascade(pl->dim, ca, reduce, st);
}

extern "C" int fvb_plan_create(int flavour, int dim, int p, int64_t T, int chunks, fvb_plan** out) {
    if (out == nullptr) return fail(FVB_EINVAL, "null plan output");
    *out = nullptr;
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    if (flavour != FVB_FUSED && flavour != FVB_CASCADE && flavour != FVB_GRAPH)
        return fail(FVB_EINVAL, "unknown flavour %d", flavour);
    if (chunks < 1) chunks = 1;
    if (chunks > T) chunks = (int)T;
    if (flavour == FVB_FUSED && (rc = fused_fits(dim, p))) return rc;
    std::unique_ptr<fvb_plan> pl(new fvb_plan());
    pl->flavour = flavour, pl->dim = dim, pl->p = p, pl->T = T, pl->chunks = chunks;
    pl->physics = physics();
    if (flavour != FVB_FUSED && (rc = alloc_scratch(pl.get()))) return rc;
    *out = pl.release();
    return FVB_OK;
}

extern "C" int fvb_scratch_doubles(int dim, int p, int64_t T, int64_t* flux_doubles,
                                   int64_t* lambda_doubles) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    const long long R = (p + 2) * ipow_h(p, dim - 1);
    if (flux_doubles) *flux_doubles = (int64_t)(dim + 2) * T * R;
    if (lambda_doubles) *lambda_doubles = (int64_t)T * R;
    return FVB_OK;
}

extern "C" int fvb_plan_create_ext(int flavour, int dim, int p, int64_t T, int chunks,
                                   double* const* flux_dev, double* const* lambda_dev, fvb_plan** out) {
    if (out == nullptr) return fail(FVB_EINVAL, "null plan output");
    *out = nullptr;
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    if (flavour != FVB_FUSED && flavour != FVB_CASCADE && flavour != FVB_GRAPH)
        return fail(FVB_EINVAL, "unknown flavour %d", flavour);
    if (flavour != FVB_FUSED && (flux_dev == nullptr || lambda_dev == nullptr))
        return fail(FVB_EINVAL, "the cascade / graph flavours need flux and wave-speed temporaries");
    if (chunks < 1) chunks = 1;
    if (chunks > T) chunks = (int)T;
    if (flavour == FVB_FUSED && (rc = fused_fits(dim, p))) return rc;
    std::unique_ptr<fvb_plan> pl(new fvb_plan());
    pl->flavour = flavour, pl->dim = dim, pl->p = p, pl->T = T, pl->chunks = chunks;
    pl->physics = physics();
    pl->external_scratch = true;
    for (int a = 0; a < 3; ++a) {
        pl->ca.tmp_flux[a] = (flavour != FVB_FUSED && a < dim) ? flux_dev[a] : nullptr;
        pl->ca.tmp_lam[a] = (flavour != FVB_FUSED && a < dim) ? lambda_dev[a] : nullptr;
        if (flavour != FVB_FUSED && a < dim && (pl->ca.tmp_flux[a] == nullptr || pl->ca.tmp_lam[a] == nullptr))
            return fail(FVB_EINVAL, "null temporary for axis %d", a);
    }
    *out = pl.release();
    return FVB_OK;
}

extern "C" int fvb_plan_execute(fvb_plan* plan, const double* q_in_dev, double* q_out_dev,
                                double dt, double h, double gamma, int with_reduction,
                                double* lam_dev, double* lam_patch_dev, void* stream) {
    if (plan == nullptr) return fail(FVB_EINVAL, "null plan");
    return plan_run(plan, q_in_dev, q_out_dev, dt, h, gamma, with_reduction, lam_dev,
                    lam_patch_dev, (cudaStream_t)stream);
}

extern "C" int fvb_plan_execute_ex(fvb_plan* plan, const double* q_in_dev, double* q_out_dev,
                                   const double* const* in_tab_dev, double* const* out_tab_dev,
                                   int64_t t0, int64_t t1, int zero_outputs, double dt, double h,
                                   double gamma, int with_reduction, double* lam_dev,
                                   double* lam_patch_dev, void* stream) {
    if (plan == nullptr) return fail(FVB_EINVAL, "null plan");
    RunOpts o;
    o.in_tab = in_tab_dev, o.out_tab = out_tab_dev;
    o.t0 = t0, o.t1 = t1, o.zero = zero_outputs != 0;
    return plan_run(plan, q_in_dev, q_out_dev, dt, h, gamma, with_reduction, lam_dev, lam_patch_dev,
                    (cudaStream_t)stream, o);
}

extern "C" int fvb_plan_graph_nodes(const fvb_plan* plan, int64_t* nodes) {
    if (plan == nullptr || nodes == nullptr) return fail(FVB_EINVAL, "null argument");
    int64_t n = 0;
    for (int r = 0; r < 2; ++r)
        for (int l = 0; l < 2; ++l)
            if (plan->graph_nodes[r][l] > n) n = plan->graph_nodes[r][l];
    *nodes = n;
    return FVB_OK;
}

extern "C" int fvb_plan_kernel_launches(const fvb_plan* plan, int with_reduction, int64_t* launches) {
    if (plan == nullptr || launches == nullptr) return fail(FVB_EINVAL, "null argument");
    const int steps = 1 + 3 * plan->dim + (with_reduction ? 1 : 0);
    if (plan->flavour == FVB_FUSED) *launches = 1;
    else if (plan->flavour == FVB_CASCADE) *launches = steps;
    else {
        long long nonempty = plan->chunks < plan->T ? plan->chunks : plan->T;
        *launches = nonempty * steps;
    }
    return FVB_OK;
}

extern "C" int fvb_plan_destroy(fvb_plan* plan) {
    if (plan == nullptr) return FVB_OK;
    for (int r = 0; r < 2; ++r)
        for (int l = 0; l < 2; ++l) {
            if (plan->exec[r][l]) cudaGraphExecDestroy(plan->exec[r][l]);
            if (plan->graph[r][l]) cudaGraphDestroy(plan->graph[r][l]);
        }
    if (plan->scratch && !plan->external_scratch) cudaFree(plan->scratch);
    delete plan;
    return FVB_OK;
}

extern "C" int fvb_plan_set_layout(fvb_plan* plan, int layout) {
    if (plan == nullptr) return fail(FVB_EINVAL, "null plan");
    if (layout != FVB_LAYOUT_AOS && layout != FVB_LAYOUT_SOA && layout != FVB_LAYOUT_AOSOA)
        return fail(FVB_EINVAL, "unknown layout %d", layout);
    plan->layout = layout;
    return FVB_OK;
}

// Cached plans for fvb_step, keyed by (device, flavour, dim, p, T, stream,
// physics, stream_thread_key): a plan owns the scratch its launches use.
// A cached plan is shared by every host thread stepping that key, so each
// run holds the plan's mutex from the layout assignment through the launch
// (the graph flavour rebinds the instantiated graph's node parameters).
static std::mutex g_cache_mu;
static std::map<std::tuple<int, int, int, int, long long, void*, int, size_t>, fvb_plan*> g_cache;

extern "C" int fvb_step(int flavour, int dim, int p, int64_t T, const double* q_in_dev,
                        double* q_out_dev, double dt, double h, double gamma, int with_reduction,
                        double* lam_dev, double* lam_patch_dev, void* stream) {
    return fvb_step_layout(flavour, FVB_LAYOUT_SOA, dim, p, T, q_in_dev, q_out_dev, dt, h, gamma,
                           with_reduction, lam_dev, lam_patch_dev, stream);
}

static int step_any(int flavour, int layout, int dim, int p, int64_t T, const double* q_in_dev,
                    double* q_out_dev, double dt, double h, double gamma, int with_reduction,
                    double* lam_dev, double* lam_patch_dev, void* stream, const RunOpts& o) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    if (layout != FVB_LAYOUT_AOS && layout != FVB_LAYOUT_SOA && layout != FVB_LAYOUT_AOSOA)
        return fail(FVB_EINVAL, "unknown layout %d", layout);
    if (flavour == FVB_FUSED) {  // stateless: no arena, no cache
        if ((rc = fused_fits(dim, p))) return rc;
        fvb_plan tmp;
        tmp.flavour = FVB_FUSED, tmp.dim = dim, tmp.p = p, tmp.T = T, tmp.chunks = 1;
        tmp.layout = layout;
        tmp.physics = physics();
        return plan_run(&tmp, q_in_dev, q_out_dev, dt, h, gamma, with_reduction, lam_dev,
                        lam_patch_dev, (cudaStream_t)stream, o);
    }
    fvb_plan* pl = nullptr;
    const RelaxedCapture relaxed;  // plan scratch / task graph built eagerly inside a user's capture
    {
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto key = std::make_tuple(dev, flavour, dim, p, (long long)T, stream, physics(), stream_thread_key(stream));
        auto it = g_cache.find(key);
        if (it != g_cache.end()) {
            pl = it->second;
        } else {
            if ((rc = fvb_plan_create(flavour, dim, p, T, 1, &pl))) return rc;
            g_cache[key] = pl;
        }
    }
    std::lock_guard<std::mutex> run_lock(pl->mu);
    pl->layout = layout;
    return plan_run(pl, q_in_dev, q_out_dev, dt, h, gamma, with_reduction, lam_dev, lam_patch_dev,
                    (cudaStream_t)stream, o);
}

extern "C" int fvb_step_layout(int flavour, int layout, int dim, int p, int64_t T,
                               const double* q_in_dev, double* q_out_dev, double dt, double h,
                               double gamma, int with_reduction, double* lam_dev,
                               double* lam_patch_dev, void* stream) {
    return step_any(flavour, layout, dim, p, T, q_in_dev, q_out_dev, dt, h, gamma, with_reduction,
                    lam_dev, lam_patch_dev, stream, RunOpts());
}

extern "C" int fvb_step_range(int flavour, int layout, int dim, int p, int64_t T, int64_t t0,
                              int64_t t1, const double* q_in_dev, double* q_out_dev, double dt,
                              double h, double gamma, int with_reduction, int zero_outputs,
                              double* lam_dev, double* lam_patch_dev, void* stream) {
    if (flavour == FVB_GRAPH) return fail(FVB_EINVAL, "fvb_step_range: the task graph runs whole batches");
    RunOpts o;
    o.t0 = t0, o.t1 = t1, o.zero = zero_outputs != 0;
    if (t1 <= t0) return fail(FVB_EINVAL, "empty patch range [%lld, %lld)", (long long)t0, (long long)t1);
    return step_any(flavour, layout, dim, p, T, q_in_dev, q_out_dev, dt, h, gamma, with_reduction,
                    lam_dev, lam_patch_dev, stream, o);
}

extern "C" int fvb_step_table(int flavour, int dim, int p, int64_t T, const double* const* in_tab_dev,
                              double* const* out_tab_dev, double dt, double h, double gamma,
                              int with_reduction, double* lam_dev, double* lam_patch_dev, void* stream) {
    if (in_tab_dev == nullptr || out_tab_dev == nullptr) return fail(FVB_EINVAL, "null pointer table");
    RunOpts o;
    o.in_tab = in_tab_dev, o.out_tab = out_tab_dev;
    return step_any(flavour, FVB_LAYOUT_AOS, dim, p, T, nullptr, nullptr, dt, h, gamma, with_reduction,
                    lam_dev, lam_patch_dev, stream, o);
}

extern "C" int fvb_step_lts(int flavour, int layout, int dim, int p, int64_t T, const double* q_in_dev,
                            double* q_out_dev, const double* dt_patch_dev, double h, double gamma,
                            int with_reduction, double* lam_dev, double* lam_patch_dev, void* stream) {
    if (dt_patch_dev == nullptr) return fail(FVB_EINVAL, "fvb_step_lts needs dt_patch_dev");
    RunOpts o;
    o.dt_patch = dt_patch_dev;
    return step_any(flavour, layout, dim, p, T, q_in_dev, q_out_dev, 0.0, h, gamma, with_reduction,
                    lam_dev, lam_patch_dev, stream, o);
}

extern "C" int fvb_step_dt(int flavour, int layout, int dim, int p, int64_t T, const double* q_in_dev,
                           double* q_out_dev, const double* dt_dev, double h, double gamma,
                           int with_reduction, double* lam_dev, double* lam_patch_dev, void* stream) {
    if (dt_dev == nullptr) return fail(FVB_EINVAL, "fvb_step_dt needs dt_dev");
    RunOpts o;
    o.dt_dev = dt_dev;
    return step_any(flavour, layout, dim, p, T, q_in_dev, q_out_dev, 0.0, h, gamma, with_reduction,
                    lam_dev, lam_patch_dev, stream, o);
}

extern "C" int fvb_release_all(void) {
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (auto& kv : g_cache) fvb_plan_destroy(kv.second);
        g_cache.clear();
    }
    // reduction slots: freed after the device drained (made and zeroed
    // again on next use, so a launch that died mid-way cannot leave a
    // stale maximum behind)
    std::lock_guard<std::mutex> lk(g_slot_mu);
    if (!g_slots.empty()) {
        cudaDeviceSynchronize();
        for (auto& kv : g_slots) cudaFree(kv.second);
        g_slots.clear();
        cudaGetLastError();
    }
    return FVB_OK;
}

