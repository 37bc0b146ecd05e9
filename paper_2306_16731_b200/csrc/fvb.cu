// fvb.cu -- libfvb.so: the C ABI declared in include/fvb.h.
//
// Host-side dispatch of the three realisation flavours (fused / cascade /
// CUDA-graph), the scratch arena + graph cache, the seeded field generator,
// the AoS<->SoA transfer kernels and the microkernel probe.  No torch types:
// plain pointers, sizes and a cudaStream_t.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false
// (no FMA contraction: bit parity with the numpy/Python reference).

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/fvb.h"
#include "cascade.cuh"
#include "common.cuh"
#include "euler.cuh"
#include "fused2d.cuh"
#include "fused_generic.cuh"

using namespace fvb;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;

static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define FVB_CUDA(call)                                                                       \
    do {                                                                                      \
        cudaError_t _e = (call);                                                              \
        if (_e != cudaSuccess)                                                                \
            return fail(FVB_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e),   \
                        __FILE__, __LINE__);                                                  \
    } while (0)

static int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(FVB_ECUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
    return FVB_OK;
}

extern "C" const char* fvb_version(void) { return "fvb 0.1.0 sm_100a"; }
extern "C" const char* fvb_last_error(void) { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// shapes
// ---------------------------------------------------------------------------
static long long ipow_h(long long b, int e) {
    long long r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

static int validate_shape(int dim, int p, int64_t T) {
    if (dim != 2 && dim != 3) return fail(FVB_EINVAL, "dim must be 2 or 3, got %d", dim);
    if (p < 2) return fail(FVB_EINVAL, "patch_size must be >= 2, got %d", p);
    if (T < 1) return fail(FVB_EINVAL, "patch_count must be >= 1, got %lld", (long long)T);
    if (ipow_h(p + 2, dim) > (1LL << 30)) return fail(FVB_EINVAL, "patch too large (p=%d)", p);
    return FVB_OK;
}

static int validate_run(double dt, double h, double gamma) {
    if (!(dt > 0.0)) return fail(FVB_EINVAL, "dt must be positive, got %g", dt);
    if (!(h > 0.0)) return fail(FVB_EINVAL, "h must be positive, got %g", h);
    if (!(gamma > 1.0)) return fail(FVB_EINVAL, "adiabatic exponent must exceed 1, got %g", gamma);
    return FVB_OK;
}

static int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

static int smem_optin() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (n <= 0) n = 227 * 1024;
    }
    return n;
}

static long long blocks_for(long long work, int threads, int per_sm) {
    long long b = (work + threads - 1) / threads;
    long long cap = (long long)sm_count() * per_sm;
    if (b > cap) b = cap;
    return b < 1 ? 1 : b;
}

// ---------------------------------------------------------------------------
// fused flavour
// ---------------------------------------------------------------------------
static constexpr int kPencilWarps = 4;
static constexpr int kGenericThreads = 256;

template <int P, bool R>
static int launch_pencil_p(const StepArgs& a, cudaStream_t st) {
    auto kern = fused2d_pencil_kernel<P, kPencilWarps, R>;
    static int occ = 0;
    if (occ == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kPencilWarps * 32, 0);
        if (occ <= 0) occ = 1;
    }
    constexpr int G = 32 / P;
    const long long groups = (a.t1 - a.t0 + G - 1) / G;
    long long blocks = (groups + kPencilWarps - 1) / kPencilWarps;
    const long long cap = (long long)sm_count() * occ;
    if (blocks > cap) blocks = cap;
    kern<<<(unsigned)blocks, kPencilWarps * 32, 0, st>>>(a);
    return check_launch("fused2d_pencil_kernel");
}

template <bool R>
static int launch_pencil(const StepArgs& a, cudaStream_t st) {
    switch (a.p) {
#define FVB_P(PP) \
    case PP:      \
        return launch_pencil_p<PP, R>(a, st);
        FVB_P(2) FVB_P(3) FVB_P(4) FVB_P(5) FVB_P(6) FVB_P(7) FVB_P(8) FVB_P(9) FVB_P(10)
        FVB_P(11) FVB_P(12) FVB_P(13) FVB_P(14) FVB_P(15) FVB_P(16) FVB_P(17) FVB_P(18)
        FVB_P(19) FVB_P(20) FVB_P(21) FVB_P(22) FVB_P(23) FVB_P(24) FVB_P(25) FVB_P(26)
        FVB_P(27) FVB_P(28) FVB_P(29) FVB_P(30) FVB_P(31) FVB_P(32)
#undef FVB_P
        default:
            return fail(FVB_EINVAL, "pencil kernel has no instance for p=%d", a.p);
    }
}

static long long generic_smem_bytes(int dim, int p) { return generic_smem_doubles(dim, p) * 8; }

template <int D, bool R>
static int launch_generic(const StepArgs& a, cudaStream_t st) {
    auto kern = fused_generic_kernel<D, kGenericThreads, R>;
    const long long smem = generic_smem_bytes(D, a.p);
    if (smem > smem_optin())
        return fail(FVB_ELIMIT,
                    "(p+2)^d staging for d=%d p=%d needs %lld B shared memory > %d B per CTA; "
                    "use the cascade or graph flavour",
                    D, a.p, smem, smem_optin());
    static int configured = 0;
    if (!configured) {
        FVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin()));
        configured = 1;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGenericThreads, (size_t)smem);
    if (occ <= 0) occ = 1;
    long long blocks = a.t1 - a.t0;
    const long long cap = (long long)sm_count() * occ;
    if (blocks > cap) blocks = cap;
    kern<<<(unsigned)blocks, kGenericThreads, (size_t)smem, st>>>(a);
    return check_launch("fused_generic_kernel");
}

static bool uses_pencil(int dim, int p) { return dim == 2 && p <= 32; }

static int launch_fused(int dim, const StepArgs& a, bool reduce, cudaStream_t st) {
    if (uses_pencil(dim, a.p)) return reduce ? launch_pencil<true>(a, st) : launch_pencil<false>(a, st);
    if (dim == 2) return reduce ? launch_generic<2, true>(a, st) : launch_generic<2, false>(a, st);
    return reduce ? launch_generic<3, true>(a, st) : launch_generic<3, false>(a, st);
}

extern "C" int fvb_fused_limit(int dim, int* max_p) {
    if (dim != 2 && dim != 3) return fail(FVB_EINVAL, "dim must be 2 or 3, got %d", dim);
    int p = 2;
    while (generic_smem_bytes(dim, p + 1) <= smem_optin() || uses_pencil(dim, p + 1)) ++p;
    *max_p = p;
    return FVB_OK;
}

extern "C" int fvb_fused_smem_bytes(int dim, int p, int64_t* bytes) {
    int rc = validate_shape(dim, p, 1);
    if (rc) return rc;
    *bytes = uses_pencil(dim, p) ? (int64_t)(2 * kPencilWarps * 4 * 32 * 8) : generic_smem_bytes(dim, p);
    return FVB_OK;
}

// ---------------------------------------------------------------------------
// cascade flavour and plans
// ---------------------------------------------------------------------------
static constexpr int kEltThreads = 256;
static constexpr int kReduceThreads = 256;

struct KernelLaunch {
    void* func;
    dim3 grid, block;
    std::vector<uint8_t> args;  // packed argument storage
    std::vector<void*> argv;
    std::vector<int> deps;      // indices into plan node list
};

struct fvb_plan {
    int flavour, dim, p, chunks;
    long long T;
    double* scratch = nullptr;  // flux + lambda temporaries (cascade / graph)
    size_t scratch_bytes = 0;
    CascadeArgs ca{};
    // graph flavour: one instantiated graph per (with_reduction, has_lam_patch)
    cudaGraphExec_t exec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
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

// kernel function pointers of the cascade steps
struct CascadeFns {
    void *copy, *flux, *lam, *acc, *reduce;
};
static CascadeFns cascade_fns(int dim) {
    if (dim == 2)
        return {(void*)cascade_copy_kernel<2>, (void*)cascade_flux_kernel<2, false>,
                (void*)cascade_flux_kernel<2, true>, (void*)cascade_acc_kernel<2>,
                (void*)cascade_reduce_kernel<2, kReduceThreads>};
    return {(void*)cascade_copy_kernel<3>, (void*)cascade_flux_kernel<3, false>,
            (void*)cascade_flux_kernel<3, true>, (void*)cascade_acc_kernel<3>,
            (void*)cascade_reduce_kernel<3, kReduceThreads>};
}

static int launch_cascade(fvb_plan* pl, const StepArgs& a, bool reduce, cudaStream_t st) {
    CascadeArgs ca = pl->ca;
    ca.s = a;
    const int d = pl->dim;
    const long long span = a.t1 - a.t0;
    const long long Mi = ipow_h(a.p, d), R = (a.p + 2) * ipow_h(a.p, d - 1);
    const unsigned gi = (unsigned)blocks_for(span * Mi, kEltThreads, 16);
    const unsigned gr = (unsigned)blocks_for(span * R, kEltThreads, 16);
    if (d == 2) {
        cascade_copy_kernel<2><<<gi, kEltThreads, 0, st>>>(a);
        for (int ax = 0; ax < 2; ++ax) cascade_flux_kernel<2, false><<<gr, kEltThreads, 0, st>>>(ca, ax);
        for (int ax = 0; ax < 2; ++ax) cascade_flux_kernel<2, true><<<gr, kEltThreads, 0, st>>>(ca, ax);
        for (int ax = 0; ax < 2; ++ax) cascade_acc_kernel<2><<<gi, kEltThreads, 0, st>>>(ca, ax);
        if (reduce) cascade_reduce_kernel<2, kReduceThreads><<<gi, kReduceThreads, 0, st>>>(a);
    } else {
        cascade_copy_kernel<3><<<gi, kEltThreads, 0, st>>>(a);
        for (int ax = 0; ax < 3; ++ax) cascade_flux_kernel<3, false><<<gr, kEltThreads, 0, st>>>(ca, ax);
        for (int ax = 0; ax < 3; ++ax) cascade_flux_kernel<3, true><<<gr, kEltThreads, 0, st>>>(ca, ax);
        for (int ax = 0; ax < 3; ++ax) cascade_acc_kernel<3><<<gi, kEltThreads, 0, st>>>(ca, ax);
        if (reduce) cascade_reduce_kernel<3, kReduceThreads><<<gi, kReduceThreads, 0, st>>>(a);
    }
    return check_launch("cascade kernels");
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
    const CascadeFns fns = cascade_fns(d);
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
    cudaGraphDestroy(g);
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
        b.lam_bits == a.lam_bits && b.lam_patch == a.lam_patch)
        return FVB_OK;
    // memset destinations changed -> rebuild; kernel args -> in-place update
    if (b.lam_bits != a.lam_bits || b.lam_patch != a.lam_patch) {
        cudaGraphExecDestroy(pl->exec[ri][li]);
        pl->exec[ri][li] = nullptr;
        return build_graph(pl, a, reduce, has_lp);
    }
    const CascadeFns fns = cascade_fns(pl->dim);
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
    }
    pl->bound[ri][li] = a;
    return FVB_OK;
}

static int plan_run(fvb_plan* pl, const double* q_in, double* q_out, double dt, double h,
                    double gamma, int with_reduction, double* lam, double* lam_patch,
                    cudaStream_t st) {
    int rc = validate_run(dt, h, gamma);
    if (rc) return rc;
    if (q_in == nullptr || q_out == nullptr) return fail(FVB_EINVAL, "null batch pointer");
    const bool reduce = with_reduction != 0;
    if (reduce && lam == nullptr) return fail(FVB_EINVAL, "with_reduction needs lam_dev");
    StepArgs a{};
    a.q_in = q_in;
    a.q_out = q_out;
    a.T = pl->T;
    a.t0 = 0;
    a.t1 = pl->T;
    a.scale = dt / h;
    a.gamma = gamma;
    a.lam_bits = reduce ? reinterpret_cast<unsigned long long*>(lam) : nullptr;
    a.lam_patch = reduce ? lam_patch : nullptr;
    a.p = pl->p;
    const bool has_lp = a.lam_patch != nullptr;
    if (pl->flavour == FVB_GRAPH) {
        const int ri = reduce ? 1 : 0, li = has_lp ? 1 : 0;
        if (pl->exec[ri][li] == nullptr) {
            if ((rc = build_graph(pl, a, reduce, has_lp))) return rc;
        } else if ((rc = rebind_graph(pl, a, reduce, has_lp))) {
            return rc;
        }
        FVB_CUDA(cudaGraphLaunch(pl->exec[ri][li], st));
        return FVB_OK;
    }
    if (reduce) {
        FVB_CUDA(cudaMemsetAsync(lam, 0, sizeof(double), st));
        if (has_lp) FVB_CUDA(cudaMemsetAsync(lam_patch, 0, sizeof(double) * pl->T, st));
    }
    if (pl->flavour == FVB_FUSED) return launch_fused(pl->dim, a, reduce, st);
    return launch_cascade(pl, a, reduce, st);
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
    if (flavour == FVB_FUSED && !uses_pencil(dim, p) && generic_smem_bytes(dim, p) > smem_optin())
        return fail(FVB_ELIMIT,
                    "(p+2)^d staging for d=%d p=%d needs %lld B shared memory > %d B per CTA; "
                    "use the cascade or graph flavour",
                    dim, p, generic_smem_bytes(dim, p), smem_optin());
    std::unique_ptr<fvb_plan> pl(new fvb_plan());
    pl->flavour = flavour, pl->dim = dim, pl->p = p, pl->T = T, pl->chunks = chunks;
    if (flavour != FVB_FUSED && (rc = alloc_scratch(pl.get()))) return rc;
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
        for (int l = 0; l < 2; ++l)
            if (plan->exec[r][l]) cudaGraphExecDestroy(plan->exec[r][l]);
    if (plan->scratch) cudaFree(plan->scratch);
    delete plan;
    return FVB_OK;
}

// cached plans for fvb_step, keyed by (flavour, dim, p, T, stream)
static std::mutex g_cache_mu;
static std::map<std::tuple<int, int, int, long long, void*>, fvb_plan*> g_cache;

extern "C" int fvb_step(int flavour, int dim, int p, int64_t T, const double* q_in_dev,
                        double* q_out_dev, double dt, double h, double gamma, int with_reduction,
                        double* lam_dev, double* lam_patch_dev, void* stream) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    if (flavour == FVB_FUSED) {  // stateless: no arena, no cache
        if (!uses_pencil(dim, p) && generic_smem_bytes(dim, p) > smem_optin())
            return fail(FVB_ELIMIT,
                        "(p+2)^d staging for d=%d p=%d needs %lld B shared memory > %d B per CTA; "
                        "use the cascade or graph flavour",
                        dim, p, generic_smem_bytes(dim, p), smem_optin());
        fvb_plan tmp;
        tmp.flavour = FVB_FUSED, tmp.dim = dim, tmp.p = p, tmp.T = T, tmp.chunks = 1;
        return plan_run(&tmp, q_in_dev, q_out_dev, dt, h, gamma, with_reduction, lam_dev,
                        lam_patch_dev, (cudaStream_t)stream);
    }
    fvb_plan* pl = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto key = std::make_tuple(flavour, dim, p, (long long)T, stream);
        auto it = g_cache.find(key);
        if (it != g_cache.end()) {
            pl = it->second;
        } else {
            if ((rc = fvb_plan_create(flavour, dim, p, T, 1, &pl))) return rc;
            g_cache[key] = pl;
        }
    }
    return plan_run(pl, q_in_dev, q_out_dev, dt, h, gamma, with_reduction, lam_dev, lam_patch_dev,
                    (cudaStream_t)stream);
}

extern "C" int fvb_release_all(void) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (auto& kv : g_cache) fvb_plan_destroy(kv.second);
    g_cache.clear();
    return FVB_OK;
}

// ---------------------------------------------------------------------------
// seeded field (bench.py:89-133)
// ---------------------------------------------------------------------------
#define FVB_LCG_A 6364136223846793005ULL
#define FVB_LCG_C 1442695040888963407ULL

__device__ __forceinline__ unsigned long long lcg_jump(unsigned long long s, unsigned long long n) {
    unsigned long long acc_a = 1, acc_c = 0, a = FVB_LCG_A, c = FVB_LCG_C;
    while (n) {
        if (n & 1) {
            acc_a *= a;
            acc_c = acc_c * a + c;
        }
        c = (a + 1) * c;
        a *= a;
        n >>= 1;
    }
    return acc_a * s + acc_c;
}

__device__ __forceinline__ double lcg_uniform(unsigned long long& s, double lo, double hi) {
    s = s * FVB_LCG_A + FVB_LCG_C;
    return lo + (hi - lo) * ((double)(s >> 11) * 0x1p-53);
}

template <int D>
__global__ void init_field_kernel(long long T, long long p0, int p, unsigned long long seed,
                                  double gamma, double* __restrict__ q) {
    constexpr int N = D + 2;
    const long long M = ipow_d(p + 2, D);
    const long long total = T * M;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long patch = i / M, lin = i - patch * M;
        unsigned long long s = lcg_jump(seed, (unsigned long long)(((p0 + patch) * M + lin) * N));
        const double rho = lcg_uniform(s, 0.5, 2.0);
        double u[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < D; ++k) u[k] = lcg_uniform(s, -0.5, 0.5);
        const double pr = lcg_uniform(s, 0.5, 2.0);
        double ke = u[0] * u[0] + u[1] * u[1];
        if (D == 3) ke = ke + u[2] * u[2];
        q[i] = rho;
#pragma unroll
        for (int k = 0; k < D; ++k) q[(1 + k) * total + i] = rho * u[k];
        q[(D + 1) * total + i] = pr / (gamma - 1.0) + 0.5 * rho * ke;
    }
}

extern "C" int fvb_init_field(int dim, int p, int64_t T_local, int64_t patch_begin, uint64_t seed,
                              double gamma, double* q_in_dev, void* stream) {
    int rc = validate_shape(dim, p, T_local);
    if (rc) return rc;
    if (patch_begin < 0) return fail(FVB_EINVAL, "patch_begin must be >= 0");
    const long long total = T_local * ipow_h(p + 2, dim);
    const unsigned grid = (unsigned)blocks_for(total, 256, 16);
    if (dim == 2)
        init_field_kernel<2><<<grid, 256, 0, (cudaStream_t)stream>>>(T_local, patch_begin, p, seed, gamma, q_in_dev);
    else
        init_field_kernel<3><<<grid, 256, 0, (cudaStream_t)stream>>>(T_local, patch_begin, p, seed, gamma, q_in_dev);
    return check_launch("init_field_kernel");
}

// ---------------------------------------------------------------------------
// AoS <-> SoA (memory.py:240-265)
// ---------------------------------------------------------------------------
__global__ void aos_soa_kernel(long long T, long long M, int N, const double* __restrict__ src,
                               double* __restrict__ dst, int to_soa) {
    const long long total = T * M * N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        // i enumerates the SoA array: k slowest, then patch, then lin
        const long long k = i / (T * M), rest = i - k * T * M;  // rest = patch*M + lin
        const long long j = rest * N + k;                          // AoS offset
        if (to_soa) dst[i] = __ldg(src + j);
        else dst[j] = __ldg(src + i);
    }
}

static int aos_soa(int dim, int p, int64_t T, int haloed, const double* src, double* dst,
                   void* stream, int to_soa) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    const long long m = haloed ? p + 2 : p, M = ipow_h(m, dim);
    const long long total = T * M * (dim + 2);
    aos_soa_kernel<<<(unsigned)blocks_for(total, 256, 16), 256, 0, (cudaStream_t)stream>>>(
        T, M, dim + 2, src, dst, to_soa);
    return check_launch("aos_soa_kernel");
}

extern "C" int fvb_aos_to_soa(int dim, int p, int64_t T, int haloed, const double* aos_dev,
                              double* soa_dev, void* stream) {
    return aos_soa(dim, p, T, haloed, aos_dev, soa_dev, stream, 1);
}

extern "C" int fvb_soa_to_aos(int dim, int p, int64_t T, int haloed, const double* soa_dev,
                              double* aos_dev, void* stream) {
    return aos_soa(dim, p, T, haloed, soa_dev, aos_dev, stream, 0);
}

// ---------------------------------------------------------------------------
// microkernel probe + admissibility
// ---------------------------------------------------------------------------
template <int D>
__global__ void microkernel_probe_kernel(long long count, int axis, double gamma,
                                         const double* __restrict__ q, double* __restrict__ f,
                                         double* __restrict__ lam) {
    constexpr int N = D + 2;
    const Euler<D> eq{gamma};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        double s[N], fl[N];
#pragma unroll
        for (int k = 0; k < N; ++k) s[k] = q[i * N + k];
        eq.flux(s, axis, fl);
#pragma unroll
        for (int k = 0; k < N; ++k) f[i * N + k] = fl[k];
        lam[i] = eq.max_eigenvalue(s, axis);
    }
}

extern "C" int fvb_eval_microkernels(int dim, int64_t count, int axis, double gamma,
                                     const double* q_dev, double* flux_dev, double* lambda_dev,
                                     void* stream) {
    if (dim != 2 && dim != 3) return fail(FVB_EINVAL, "dim must be 2 or 3, got %d", dim);
    if (axis < 0 || axis >= dim) return fail(FVB_EINVAL, "axis %d out of range for d=%d", axis, dim);
    if (count < 0) return fail(FVB_EINVAL, "negative count");
    if (count == 0) return FVB_OK;
    const unsigned grid = (unsigned)blocks_for(count, 256, 16);
    if (dim == 2)
        microkernel_probe_kernel<2><<<grid, 256, 0, (cudaStream_t)stream>>>(count, axis, gamma, q_dev, flux_dev, lambda_dev);
    else
        microkernel_probe_kernel<3><<<grid, 256, 0, (cudaStream_t)stream>>>(count, axis, gamma, q_dev, flux_dev, lambda_dev);
    return check_launch("microkernel_probe_kernel");
}

template <int D>
__global__ void admissible_kernel(long long T, long long M, double gamma,
                                  const double* __restrict__ q, unsigned long long* __restrict__ bad) {
    constexpr int N = D + 2;
    const Euler<D> eq{gamma};
    const long long total = T * M;
    unsigned long long local = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        double s[N];
#pragma unroll
        for (int k = 0; k < N; ++k) s[k] = __ldg(q + k * total + i);
        if (!(s[0] > 0.0) || !(eq.pressure(s) > 0.0)) ++local;
    }
    if (local) atomicAdd(bad, local);
}

extern "C" int fvb_check_admissible(int dim, int p, int64_t T, int haloed, double gamma,
                                    const double* q_dev, int64_t* bad_count_dev, void* stream) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    FVB_CUDA(cudaMemsetAsync(bad_count_dev, 0, sizeof(int64_t), st));
    const long long M = ipow_h(haloed ? p + 2 : p, dim), total = T * M;
    const unsigned grid = (unsigned)blocks_for(total, 256, 16);
    auto* bad = reinterpret_cast<unsigned long long*>(bad_count_dev);
    if (dim == 2) admissible_kernel<2><<<grid, 256, 0, st>>>(T, M, gamma, q_dev, bad);
    else admissible_kernel<3><<<grid, 256, 0, st>>>(T, M, gamma, q_dev, bad);
    return check_launch("admissible_kernel");
}

extern "C" double fvb_admissible_dt(double lambda, double h, double cfl) { return cfl * h / lambda; }
