// xfer.cu -- the transfer modes of run_launch over T independently
// allocated host patches (pkg/src/patchbench/memory.py:162-265,
// bench.py:209-259), natively:
//
//   * pin manager: host ranges the GPU may address directly -- ranges we
//     registered (cudaHostRegister of the page-merged spans of a patch
//     set's arrays, refcounted, so overlapping sets share registrations)
//     and pinned blocks the caller announces (torch pinned allocations);
//   * table gather / scatter kernels: per-patch AoS arrays, addressed
//     through a device table of their (host-mapped) pointers, to / from a
//     device batch in any layout, for a patch range -- zero-copy PCIe
//     reads / writes issued by the SMs, staged through shared memory so
//     both the host side (contiguous 8-byte runs) and the batch side
//     (one unknown per warp instruction) are coalesced;
//   * fvb_launch_table: one launch.  SHARED computes in place on the
//     per-patch arrays (pointer-table kernels, no batch buffers);
//     COPY / POOLED pipeline gather(c) -> step(c) -> scatter(c) over patch
//     chunks on three streams, so PCIe reads, compute and PCIe writes of
//     different chunks overlap (the step over a chunk is bit-identical to
//     the whole-batch step: patches are independent, kernelgraph.py:215-247).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "host.h"

namespace fvb {
namespace {

// ---------------------------------------------------------------------------
// table gather / scatter kernels
// ---------------------------------------------------------------------------
constexpr int kXferThreads = 256;
constexpr int kXferWindow = 3072;  // doubles staged per window (24 KB)

// Where a patch's AoS array lives: a pointer table of per-patch arrays, or
// one contiguous block of consecutive patches (a staged chunk).
struct TableSrc {
    const double* const* tab;
    __device__ __forceinline__ const double* operator()(long long patch) const { return tab[patch]; }
};
struct TableDst {
    double* const* tab;
    __device__ __forceinline__ double* operator()(long long patch) const { return tab[patch]; }
};
struct BlockSrc {
    const double* base;  // patch `first`
    long long first, stride;
    __device__ __forceinline__ const double* operator()(long long patch) const {
        return base + (patch - first) * stride;
    }
};
struct BlockDst {
    double* base;
    long long first, stride;
    __device__ __forceinline__ double* operator()(long long patch) const { return base + (patch - first) * stride; }
};

// Haloed input: per-patch AoS arrays -> batch rows [t0, t1) in `lay`.
template <int N, class Src>
__global__ void __launch_bounds__(kXferThreads) table_gather_kernel(long long t0, long long t1, int M, Src at,
                                                                    Lay lay, double* __restrict__ dst) {
    __shared__ double win[kXferWindow];
    constexpr int W = kXferWindow / N;  // cells per window
    for (long long patch = t0 + blockIdx.x; patch < t1; patch += gridDim.x) {
        const double* __restrict__ src = at(patch);
        double* __restrict__ base = dst + patch * lay.p;
        if (lay.l == N && lay.k == 1) {  // AoS batch: the patch's array verbatim
            for (int i = threadIdx.x; i < N * M; i += kXferThreads) base[i] = src[i];
            continue;
        }
        for (int c0 = 0; c0 < M; c0 += W) {
            const int nc = min(W, M - c0);
            const double* s = src + (long long)c0 * N;
            for (int i = threadIdx.x; i < nc * N; i += kXferThreads) win[i] = s[i];
            __syncthreads();
            for (int i = threadIdx.x; i < nc * N; i += kXferThreads) {
                const int k = i / nc, c = i - k * nc;
                base[k * lay.k + (long long)(c0 + c) * lay.l] = win[c * N + k];
            }
            __syncthreads();
        }
    }
}

// Interior output: batch rows [t0, t1) in `lay` -> per-patch AoS arrays.
template <int N, class Dst>
__global__ void __launch_bounds__(kXferThreads) table_scatter_kernel(long long t0, long long t1, int M,
                                                                     const double* __restrict__ src, Lay lay,
                                                                     Dst at) {
    __shared__ double win[kXferWindow];
    constexpr int W = kXferWindow / N;
    for (long long patch = t0 + blockIdx.x; patch < t1; patch += gridDim.x) {
        double* __restrict__ out = at(patch);
        const double* __restrict__ base = src + patch * lay.p;
        if (lay.l == N && lay.k == 1) {
            for (int i = threadIdx.x; i < N * M; i += kXferThreads) out[i] = base[i];
            continue;
        }
        for (int c0 = 0; c0 < M; c0 += W) {
            const int nc = min(W, M - c0);
            for (int i = threadIdx.x; i < nc * N; i += kXferThreads) {
                const int k = i / nc, c = i - k * nc;
                win[c * N + k] = base[k * lay.k + (long long)(c0 + c) * lay.l];
            }
            __syncthreads();
            double* o = out + (long long)c0 * N;
            for (int i = threadIdx.x; i < nc * N; i += kXferThreads) o[i] = win[i];
            __syncthreads();
        }
    }
}

int valid_layout(int layout) {
    return layout == FVB_LAYOUT_AOS || layout == FVB_LAYOUT_SOA || layout == FVB_LAYOUT_AOSOA;
}

// Grids stay small (two CTAs per SM at most): the transfer kernels are PCIe
// bound and share the GPU with the step kernel of another chunk.
unsigned xfer_grid(long long patches) {
    long long cap = 2LL * sm_count();
    return (unsigned)std::max(1LL, std::min(patches, cap));
}

template <class Src>
int launch_gather_from(int dim, int p, long long T, long long t0, long long t1, Src at, int layout, double* dst,
                       cudaStream_t st, unsigned grid) {
    const int n = dim + 2;
    const long long M = ipow_h(p + 2, dim);
    const Lay lay = layout_strides(layout, T, M, n);
    if (n == 4) table_gather_kernel<4><<<grid, kXferThreads, 0, st>>>(t0, t1, (int)M, at, lay, dst);
    else table_gather_kernel<5><<<grid, kXferThreads, 0, st>>>(t0, t1, (int)M, at, lay, dst);
    return check_launch("table_gather_kernel");
}

template <class Dst>
int launch_scatter_to(int dim, int p, long long T, long long t0, long long t1, const double* src, int layout,
                      Dst at, cudaStream_t st, unsigned grid) {
    const int n = dim + 2;
    const long long M = ipow_h(p, dim);
    const Lay lay = layout_strides(layout, T, M, n);
    if (n == 4) table_scatter_kernel<4><<<grid, kXferThreads, 0, st>>>(t0, t1, (int)M, src, lay, at);
    else table_scatter_kernel<5><<<grid, kXferThreads, 0, st>>>(t0, t1, (int)M, src, lay, at);
    return check_launch("table_scatter_kernel");
}

int launch_gather(int dim, int p, long long T, long long t0, long long t1, const double* const* tab,
                  int layout, double* dst, cudaStream_t st) {
    return launch_gather_from(dim, p, T, t0, t1, TableSrc{tab}, layout, dst, st, xfer_grid(t1 - t0));
}

int launch_scatter(int dim, int p, long long T, long long t0, long long t1, const double* src, int layout,
                   double* const* tab, cudaStream_t st) {
    return launch_scatter_to(dim, p, T, t0, t1, src, layout, TableDst{tab}, st, xfer_grid(t1 - t0));
}

// Device-local permutation of a staged chunk (HBM-bound, a full grid).
unsigned stage_grid(long long patches) {
    return (unsigned)std::max(1LL, std::min(patches, 8LL * sm_count()));
}

// ---------------------------------------------------------------------------
// pin manager
// ---------------------------------------------------------------------------
struct PinEntry {
    uintptr_t end;
    int refs;
    bool ours;  // registered here (unregister at refs == 0), else announced by the caller
};
std::mutex g_pin_mu;
std::map<uintptr_t, PinEntry> g_pins;  // start -> entry; entries never overlap

constexpr uintptr_t kPage = 4096;

}  // namespace
}  // namespace fvb

using namespace fvb;

struct fvb_pin {
    std::vector<uintptr_t> held;  // starts of the entries this handle references
};

// Entries overlapping [a, b), in address order.
static std::vector<std::map<uintptr_t, PinEntry>::iterator> overlapping(uintptr_t a, uintptr_t b) {
    std::vector<std::map<uintptr_t, PinEntry>::iterator> out;
    auto it = g_pins.upper_bound(a);
    if (it != g_pins.begin()) {
        auto prev = std::prev(it);
        if (prev->second.end > a) out.push_back(prev);
    }
    for (; it != g_pins.end() && it->first < b; ++it) out.push_back(it);
    return out;
}

static void release_locked(fvb_pin* h) {
    for (uintptr_t s : h->held) {
        auto it = g_pins.find(s);
        if (it == g_pins.end()) continue;
        if (--it->second.refs == 0) {
            // a failed unregister must not leave the runtime's last error set
            // (the next torch launch check would report it as its own)
            if (it->second.ours && cudaHostUnregister(reinterpret_cast<void*>(it->first)) != cudaSuccess)
                cudaGetLastError();
            g_pins.erase(it);
        }
    }
    h->held.clear();
}

extern "C" int fvb_host_pin(const uint64_t* ptrs, int64_t count, int64_t nbytes, fvb_pin** out) {
    if (out == nullptr || (count > 0 && ptrs == nullptr) || count < 0 || nbytes <= 0)
        return fail(FVB_EINVAL, "fvb_host_pin: bad arguments");
    *out = nullptr;
    int can = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&can, cudaDevAttrCanUseHostPointerForRegisteredMem, dev);
    if (!can) return fail(FVB_ECUDA, "device %d cannot address registered host memory by its host pointer", dev);
    // page-aligned spans of the arrays, sorted and merged
    std::vector<std::pair<uintptr_t, uintptr_t>> spans;
    spans.reserve((size_t)count);
    for (int64_t i = 0; i < count; ++i) {
        const uintptr_t a = (uintptr_t)ptrs[i] & ~(kPage - 1);
        const uintptr_t b = ((uintptr_t)ptrs[i] + (uintptr_t)nbytes + kPage - 1) & ~(kPage - 1);
        spans.emplace_back(a, b);
    }
    std::sort(spans.begin(), spans.end());
    std::vector<std::pair<uintptr_t, uintptr_t>> merged;
    for (auto& s : spans) {
        if (!merged.empty() && s.first <= merged.back().second) merged.back().second = std::max(merged.back().second, s.second);
        else merged.push_back(s);
    }
    std::unique_ptr<fvb_pin> h(new fvb_pin());
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (auto& m : merged) {
        // reference what is already addressable, register the gaps between
        uintptr_t cur = m.first;
        auto hits = overlapping(m.first, m.second);
        std::vector<std::pair<uintptr_t, uintptr_t>> gaps;
        for (auto it : hits) {
            if (it->first > cur) gaps.emplace_back(cur, it->first);
            cur = std::max(cur, it->second.end);
            it->second.refs++;
            h->held.push_back(it->first);
        }
        if (cur < m.second) gaps.emplace_back(cur, m.second);
        for (auto& g : gaps) {
            cudaError_t e = cudaHostRegister(reinterpret_cast<void*>(g.first), g.second - g.first,
                                             cudaHostRegisterPortable | cudaHostRegisterMapped);
            if (e != cudaSuccess) {
                cudaGetLastError();
                release_locked(h.get());
                return fail(FVB_ECUDA, "cudaHostRegister of %zu bytes failed: %s", (size_t)(g.second - g.first),
                            cudaGetErrorString(e));
            }
            g_pins[g.first] = PinEntry{g.second, 1, true};
            h->held.push_back(g.first);
        }
    }
    *out = h.release();
    return FVB_OK;
}

extern "C" int fvb_host_note_pinned(const void* base, int64_t nbytes, fvb_pin** out) {
    if (out == nullptr || base == nullptr || nbytes <= 0) return fail(FVB_EINVAL, "fvb_host_note_pinned: bad arguments");
    *out = nullptr;
    const uintptr_t a = (uintptr_t)base, b = a + (uintptr_t)nbytes;
    std::unique_ptr<fvb_pin> h(new fvb_pin());
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!overlapping(a, b).empty()) return fail(FVB_EINVAL, "pinned block overlaps a known host range");
    g_pins[a] = PinEntry{b, 1, false};
    h->held.push_back(a);
    *out = h.release();
    return FVB_OK;
}

extern "C" int fvb_host_unpin(fvb_pin* h) {
    if (h == nullptr) return FVB_OK;
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        release_locked(h);
    }
    delete h;
    return FVB_OK;
}

// Device-addressable check of T arrays of nbytes each; *first_bad = index of
// the first array outside every known range, or -1.
static int64_t first_unpinned(const uint64_t* ptrs, int64_t count, int64_t nbytes) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto hint = g_pins.end();
    for (int64_t i = 0; i < count; ++i) {
        uintptr_t a = (uintptr_t)ptrs[i];
        const uintptr_t b = a + (uintptr_t)nbytes;
        auto it = hint;
        if (it == g_pins.end() || a < it->first || a >= it->second.end) {
            it = g_pins.upper_bound(a);
            if (it == g_pins.begin()) return i;
            --it;
            if (a >= it->second.end) return i;
        }
        hint = it;
        while (it->second.end < b) {  // the array continues into the adjacent entry
            auto nx = std::next(it);
            if (nx == g_pins.end() || nx->first != it->second.end) return i;
            it = nx;
        }
    }
    return -1;
}

// [a, a + bytes) inside ONE known range (one pinned allocation or one
// registration): a DMA may not span two registrations (cudaMemcpy fails
// with cudaErrorInvalidValue, measured).
static bool in_one_range(uintptr_t a, uint64_t bytes) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pins.upper_bound(a);
    if (it == g_pins.begin()) return false;
    --it;
    return a >= it->first && a + bytes <= it->second.end;
}

extern "C" int fvb_host_accessible(const uint64_t* ptrs, int64_t count, int64_t nbytes, int64_t* first_bad) {
    if (first_bad == nullptr || count < 0 || (count > 0 && ptrs == nullptr)) return fail(FVB_EINVAL, "bad arguments");
    *first_bad = first_unpinned(ptrs, count, nbytes);
    return FVB_OK;
}

extern "C" int fvb_gather_table(int dim, int p, int64_t T, int64_t t0, int64_t t1, const double* const* tab_dev,
                                int layout, double* batch_dev, void* stream) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    if (!valid_layout(layout)) return fail(FVB_EINVAL, "unknown layout %d", layout);
    if (t0 < 0 || t1 > T || t0 >= t1) return fail(FVB_EINVAL, "patch range [%lld, %lld)", (long long)t0, (long long)t1);
    if (tab_dev == nullptr || batch_dev == nullptr) return fail(FVB_EINVAL, "null pointer");
    return launch_gather(dim, p, T, t0, t1, tab_dev, layout, batch_dev, (cudaStream_t)stream);
}

extern "C" int fvb_scatter_table(int dim, int p, int64_t T, int64_t t0, int64_t t1, int layout,
                                 const double* batch_dev, double* const* tab_dev, void* stream) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    if (!valid_layout(layout)) return fail(FVB_EINVAL, "unknown layout %d", layout);
    if (t0 < 0 || t1 > T || t0 >= t1) return fail(FVB_EINVAL, "patch range [%lld, %lld)", (long long)t0, (long long)t1);
    if (tab_dev == nullptr || batch_dev == nullptr) return fail(FVB_EINVAL, "null pointer");
    return launch_scatter(dim, p, T, t0, t1, batch_dev, layout, tab_dev, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// fvb_launch_table: one launch of run_launch over per-patch host arrays
// ---------------------------------------------------------------------------
namespace {

struct Engine {
    int device = 0;
    cudaStream_t s_g = nullptr, s_c = nullptr, s_s = nullptr;
    uint64_t* d_in_tab = nullptr;
    uint64_t* d_out_tab = nullptr;
    // pinned copies of the caller's tables: the tables are pageable and may
    // share a page with registered patch arrays, and a pageable cudaMemcpy
    // starting inside a registered page fails (see fvb_host_pin)
    uint64_t* h_in_tab = nullptr;
    uint64_t* h_out_tab = nullptr;
    long long tab_cap = 0;
    double* d_lam = nullptr;  // one slot per chunk
    double* h_lam = nullptr;  // pinned copy of the slots
    int lam_cap = 0;
    double* d_stage_in = nullptr;   // DMA staging of one input chunk (AoS)
    double* d_stage_out = nullptr;  // and of one output chunk
    long long stage_in_cap = 0, stage_out_cap = 0;
    double* h_stage_in[2] = {nullptr, nullptr};   // pinned host chunks (host-staged path)
    double* h_stage_out[2] = {nullptr, nullptr};
    long long h_stage_in_cap = 0, h_stage_out_cap = 0;
    std::vector<cudaEvent_t> ev;  // scratch events
    std::mutex mu;                // one launch per engine at a time

    int reserve(long long T, int chunks, int events) {
        if (T > tab_cap) {
            cudaFree(d_in_tab);
            cudaFree(d_out_tab);
            cudaFreeHost(h_in_tab);
            cudaFreeHost(h_out_tab);
            d_in_tab = d_out_tab = h_in_tab = h_out_tab = nullptr;
            FVB_CUDA(cudaMalloc(&d_in_tab, sizeof(uint64_t) * T));
            FVB_CUDA(cudaMalloc(&d_out_tab, sizeof(uint64_t) * T));
            FVB_CUDA(cudaMallocHost(&h_in_tab, sizeof(uint64_t) * T));
            FVB_CUDA(cudaMallocHost(&h_out_tab, sizeof(uint64_t) * T));
            tab_cap = T;
        }
        if (chunks > lam_cap) {
            cudaFree(d_lam);
            cudaFreeHost(h_lam);
            d_lam = nullptr, h_lam = nullptr;
            FVB_CUDA(cudaMalloc(&d_lam, sizeof(double) * chunks));
            FVB_CUDA(cudaMallocHost(&h_lam, sizeof(double) * chunks));
            lam_cap = chunks;
        }
        while ((int)ev.size() < events) {
            cudaEvent_t e;
            FVB_CUDA(cudaEventCreate(&e));
            ev.push_back(e);
        }
        if (s_g == nullptr) {
            FVB_CUDA(cudaStreamCreateWithFlags(&s_g, cudaStreamNonBlocking));
            FVB_CUDA(cudaStreamCreateWithFlags(&s_c, cudaStreamNonBlocking));
            FVB_CUDA(cudaStreamCreateWithFlags(&s_s, cudaStreamNonBlocking));
        }
        return FVB_OK;
    }
    int reserve_host_stage(long long in_doubles, long long out_doubles) {
        if (in_doubles > h_stage_in_cap) {
            for (double*& b : h_stage_in) {
                cudaFreeHost(b);
                b = nullptr;
                FVB_CUDA(cudaMallocHost(&b, sizeof(double) * in_doubles));
            }
            h_stage_in_cap = in_doubles;
        }
        if (out_doubles > h_stage_out_cap) {
            for (double*& b : h_stage_out) {
                cudaFreeHost(b);
                b = nullptr;
                FVB_CUDA(cudaMallocHost(&b, sizeof(double) * out_doubles));
            }
            h_stage_out_cap = out_doubles;
        }
        return FVB_OK;
    }
    int reserve_stage(long long in_doubles, long long out_doubles) {
        if (in_doubles > stage_in_cap) {
            cudaFree(d_stage_in);
            d_stage_in = nullptr;
            FVB_CUDA(cudaMalloc(&d_stage_in, sizeof(double) * in_doubles));
            stage_in_cap = in_doubles;
        }
        if (out_doubles > stage_out_cap) {
            cudaFree(d_stage_out);
            d_stage_out = nullptr;
            FVB_CUDA(cudaMalloc(&d_stage_out, sizeof(double) * out_doubles));
            stage_out_cap = out_doubles;
        }
        return FVB_OK;
    }
};

std::mutex g_engine_mu;
// (device, caller stream, stream_thread_key): an engine's staging buffers serve its stream's launches in order
std::map<std::tuple<int, void*, size_t>, std::unique_ptr<Engine>> g_engines;

Engine* engine_for(void* stream) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_engine_mu);
    auto& e = g_engines[std::make_tuple(dev, stream, stream_thread_key(stream))];
    if (!e) {
        e.reset(new Engine());
        e->device = dev;
    }
    return e.get();
}

// A table whose entry i is entry 0 + i * bytes: the arrays are one
// contiguous host range in patch order (pinned blocks).
bool contiguous(const uint64_t* tab, int64_t T, int64_t bytes) {
    for (int64_t i = 1; i < T; ++i)
        if (tab[i] != tab[0] + (uint64_t)(i * bytes)) return false;
    return true;
}

}  // namespace

// Plans are defined in fvb.cu; the engine runs them through this entry.
extern "C" int fvb_plan_execute_ex(fvb_plan* plan, const double* q_in_dev, double* q_out_dev,
                                   const double* const* in_tab_dev, double* const* out_tab_dev,
                                   int64_t t0, int64_t t1, int zero_outputs, double dt, double h,
                                   double gamma, int with_reduction, double* lam_dev,
                                   double* lam_patch_dev, void* stream);
extern "C" int fvb_plan_create(int flavour, int dim, int p, int64_t T, int chunks, fvb_plan** out);
extern "C" int fvb_plan_destroy(fvb_plan* plan);
extern "C" int fvb_plan_set_layout(fvb_plan* plan, int layout);

extern "C" int fvb_launch_table(int flavour, int layout, int dim, int p, int64_t T, const uint64_t* in_tab_host,
                                const uint64_t* out_tab_host, double* batch_in_dev, double* batch_out_dev,
                                fvb_plan* plan, double dt, double h, double gamma, int with_reduction,
                                double* lam_patch_dev, int64_t chunk_patches, double* reduced_out,
                                double* compute_seconds_out, void* stream) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    if (!valid_layout(layout)) return fail(FVB_EINVAL, "unknown layout %d", layout);
    if (in_tab_host == nullptr || out_tab_host == nullptr) return fail(FVB_EINVAL, "null pointer table");
    const bool shared = batch_in_dev == nullptr && batch_out_dev == nullptr;
    if (!shared && (batch_in_dev == nullptr || batch_out_dev == nullptr))
        return fail(FVB_EINVAL, "COPY / POOLED launches need both batch buffers");
    if (flavour != FVB_FUSED && plan == nullptr) return fail(FVB_EINVAL, "cascade / graph launches need a plan");
    const int n = dim + 2;
    const long long nin = (long long)n * ipow_h(p + 2, dim), nout = (long long)n * ipow_h(p, dim);
    // SHARED computes on the arrays in place over PCIe: they must be
    // device-addressable (registered / pinned).  COPY / POOLED over arrays
    // that are not ("host-staged"): the host gathers each chunk into pinned
    // memory (memcpy, OpenMP threads), DMA moves it, and the reverse on the
    // way out -- the reference's host gather / scatter (memory.py:240-265)
    // feeding the copy engines, with no registration at all.
    int64_t bad = first_unpinned(in_tab_host, T, nin * 8);
    if (bad < 0) bad = first_unpinned(out_tab_host, T, nout * 8);
    if (bad >= 0 && shared)
        return fail(FVB_EINVAL, "patch %lld is not in device-addressable host memory (pin the patch set)",
                    (long long)bad);
    const bool staged = bad >= 0;
    // chunking: ~64 MB of haloed input per chunk (COPY / POOLED).  The
    // graph flavour moves its batch in chunks too but runs one whole-batch
    // step between the gathers and the scatters.
    long long cp = chunk_patches > 0 ? chunk_patches : std::max(1LL, (64LL << 20) / (nin * 8));
    if (shared) cp = T;
    cp = std::min(cp, (long long)T);
    const int chunks = (int)((T + cp - 1) / cp);
    const bool whole = flavour == FVB_GRAPH;
    // Pinned blocks (the arrays are one contiguous host range in patch
    // order, e.g. allocate_scattered(pinned=True)): chunks move by DMA on
    // the copy engines -- H2D into a staging chunk, permuted into the batch
    // layout by a device kernel, and the reverse -- instead of SM-issued
    // zero-copy PCIe reads / writes of the pointer-table kernels.  An AoS
    // batch is the host image itself: DMA straight into / out of it.  (Each
    // direction must lie in one pinned allocation or registration.)
    const bool dma = !shared && !staged && contiguous(in_tab_host, T, nin * 8) &&
                     contiguous(out_tab_host, T, nout * 8) && in_one_range(in_tab_host[0], (uint64_t)(T * nin * 8)) &&
                     in_one_range(out_tab_host[0], (uint64_t)(T * nout * 8));
    const double* h_in = reinterpret_cast<const double*>(in_tab_host[0]);
    double* h_out = reinterpret_cast<double*>(out_tab_host[0]);
    Engine* e = engine_for(stream);
    std::lock_guard<std::mutex> lk(e->mu);
    if ((rc = e->reserve(T, chunks, 3 * chunks + 7))) return rc;
    if ((dma || staged) && layout != FVB_LAYOUT_AOS && (rc = e->reserve_stage(cp * nin, cp * nout))) return rc;
    if (staged && (rc = e->reserve_host_stage(cp * nin, cp * nout))) return rc;
    // host-staged: per buffer b, [0..1] host input chunk b reusable (its H2D
    // done), [2..3] host output chunk b holds data (its D2H done)
    cudaEvent_t* hev = &e->ev[3 * chunks + 3];
    cudaStream_t st = (cudaStream_t)stream;
    cudaEvent_t ev_start = e->ev[0], ev_end = e->ev[1];
    FVB_CUDA(cudaEventRecord(ev_start, st));
    for (cudaStream_t s : {e->s_g, e->s_c, e->s_s}) FVB_CUDA(cudaStreamWaitEvent(s, ev_start, 0));
    if (!dma && !staged) {
        // the engine is held for the whole (synchronous) launch, so its
        // pinned table copies are free to overwrite here
        std::memcpy(e->h_in_tab, in_tab_host, sizeof(uint64_t) * T);
        std::memcpy(e->h_out_tab, out_tab_host, sizeof(uint64_t) * T);
        FVB_CUDA(cudaMemcpyAsync(e->d_in_tab, e->h_in_tab, sizeof(uint64_t) * T, cudaMemcpyHostToDevice, e->s_g));
        FVB_CUDA(cudaMemcpyAsync(e->d_out_tab, e->h_out_tab, sizeof(uint64_t) * T, cudaMemcpyHostToDevice, e->s_s));
    }
    const bool reduce = with_reduction != 0;
    if (reduce) {
        FVB_CUDA(cudaMemsetAsync(e->d_lam, 0, sizeof(double) * chunks, e->s_c));
        if (lam_patch_dev) FVB_CUDA(cudaMemsetAsync(lam_patch_dev, 0, sizeof(double) * T, e->s_c));
    }
    const auto* in_tab = reinterpret_cast<const double* const*>(e->d_in_tab);
    auto* out_tab = reinterpret_cast<double* const*>(e->d_out_tab);
    fvb_plan* pl = plan;
    std::unique_ptr<fvb_plan, int (*)(fvb_plan*)> tmp(nullptr, fvb_plan_destroy);
    if (pl == nullptr) {  // fused: a stateless plan
        if ((rc = fvb_plan_create(FVB_FUSED, dim, p, T, 1, &pl))) return rc;
        tmp.reset(pl);
    }
    if ((rc = fvb_plan_set_layout(pl, shared ? FVB_LAYOUT_AOS : layout))) return rc;
    // events: [0] start, [1] end, then per chunk (gather done, step start, step end)
    auto host_gather = [&](long long lo, long long hi, int b) -> int {  // patches -> pinned chunk b
        if (lo >= 2 * cp) FVB_CUDA(cudaEventSynchronize(hev[b]));  // chunk b's previous H2D is done
        double* dst = e->h_stage_in[b];
#pragma omp parallel for schedule(static)
        for (long long i = lo; i < hi; ++i)
            std::memcpy(dst + (i - lo) * nin, reinterpret_cast<const void*>(in_tab_host[i]), sizeof(double) * nin);
        return FVB_OK;
    };
    auto host_scatter = [&](long long lo, long long hi, int b) -> int {  // pinned chunk b -> patches
        FVB_CUDA(cudaEventSynchronize(hev[2 + b]));
        const double* src = e->h_stage_out[b];
#pragma omp parallel for schedule(static)
        for (long long i = lo; i < hi; ++i)
            std::memcpy(reinterpret_cast<void*>(out_tab_host[i]), src + (i - lo) * nout, sizeof(double) * nout);
        return FVB_OK;
    };
    auto gather = [&](long long lo, long long hi) -> int {
        if (staged) {
            const int b = (int)((lo / cp) & 1);
            int r = host_gather(lo, hi, b);
            if (r) return r;
            const size_t bytes = sizeof(double) * (size_t)((hi - lo) * nin);
            double* dst = layout == FVB_LAYOUT_AOS ? batch_in_dev + lo * nin : e->d_stage_in;
            FVB_CUDA(cudaMemcpyAsync(dst, e->h_stage_in[b], bytes, cudaMemcpyHostToDevice, e->s_g));
            FVB_CUDA(cudaEventRecord(hev[b], e->s_g));
            if (layout == FVB_LAYOUT_AOS) return FVB_OK;
            return launch_gather_from(dim, p, T, lo, hi, BlockSrc{e->d_stage_in, lo, nin}, layout, batch_in_dev,
                                      e->s_g, stage_grid(hi - lo));
        }
        if (!dma) return launch_gather(dim, p, T, lo, hi, in_tab, layout, batch_in_dev, e->s_g);
        const size_t bytes = sizeof(double) * (size_t)((hi - lo) * nin);
        if (layout == FVB_LAYOUT_AOS) {
            FVB_CUDA(cudaMemcpyAsync(batch_in_dev + lo * nin, h_in + lo * nin, bytes, cudaMemcpyHostToDevice, e->s_g));
            return FVB_OK;
        }
        FVB_CUDA(cudaMemcpyAsync(e->d_stage_in, h_in + lo * nin, bytes, cudaMemcpyHostToDevice, e->s_g));
        return launch_gather_from(dim, p, T, lo, hi, BlockSrc{e->d_stage_in, lo, nin}, layout, batch_in_dev, e->s_g,
                                  stage_grid(hi - lo));
    };
    auto scatter = [&](long long lo, long long hi) -> int {
        if (staged) {  // device -> pinned chunk b; host_scatter copies it out later
            const int b = (int)((lo / cp) & 1);
            const size_t bytes = sizeof(double) * (size_t)((hi - lo) * nout);
            if (layout != FVB_LAYOUT_AOS) {
                int r = launch_scatter_to(dim, p, T, lo, hi, batch_out_dev, layout, BlockDst{e->d_stage_out, lo, nout},
                                          e->s_s, stage_grid(hi - lo));
                if (r) return r;
            }
            const double* src = layout == FVB_LAYOUT_AOS ? batch_out_dev + lo * nout : e->d_stage_out;
            FVB_CUDA(cudaMemcpyAsync(e->h_stage_out[b], src, bytes, cudaMemcpyDeviceToHost, e->s_s));
            FVB_CUDA(cudaEventRecord(hev[2 + b], e->s_s));
            return FVB_OK;
        }
        if (!dma) return launch_scatter(dim, p, T, lo, hi, batch_out_dev, layout, out_tab, e->s_s);
        const size_t bytes = sizeof(double) * (size_t)((hi - lo) * nout);
        if (layout == FVB_LAYOUT_AOS) {
            FVB_CUDA(cudaMemcpyAsync(h_out + lo * nout, batch_out_dev + lo * nout, bytes, cudaMemcpyDeviceToHost, e->s_s));
            return FVB_OK;
        }
        int r = launch_scatter_to(dim, p, T, lo, hi, batch_out_dev, layout, BlockDst{e->d_stage_out, lo, nout}, e->s_s,
                                  stage_grid(hi - lo));
        if (r) return r;
        FVB_CUDA(cudaMemcpyAsync(h_out + lo * nout, e->d_stage_out, bytes, cudaMemcpyDeviceToHost, e->s_s));
        return FVB_OK;
    };
    int steps_run = 0;  // step intervals timed (events 3 + 3c, 4 + 3c)
    if (shared) {  // compute in place on the per-patch arrays: no batch, no copies
        cudaEvent_t in_ready = e->ev[2], out_ready = e->ev[3];
        FVB_CUDA(cudaEventRecord(in_ready, e->s_g));
        FVB_CUDA(cudaEventRecord(out_ready, e->s_s));
        FVB_CUDA(cudaStreamWaitEvent(e->s_c, in_ready, 0));
        FVB_CUDA(cudaStreamWaitEvent(e->s_c, out_ready, 0));
        FVB_CUDA(cudaEventRecord(e->ev[3], e->s_c));
        if ((rc = fvb_plan_execute_ex(pl, nullptr, nullptr, in_tab, out_tab, 0, -1, 1, dt, h, gamma, with_reduction,
                                      e->d_lam, lam_patch_dev, e->s_c)))
            return rc;
        FVB_CUDA(cudaEventRecord(e->ev[4], e->s_c));
        steps_run = 1;
    } else if (whole) {  // graph: every chunk in, one whole-batch step, every chunk out
        for (int c = 0; c < chunks; ++c) {
            const long long lo = (long long)c * cp, hi = std::min((long long)T, lo + cp);
            if ((rc = gather(lo, hi))) return rc;
        }
        FVB_CUDA(cudaEventRecord(e->ev[2], e->s_g));
        FVB_CUDA(cudaStreamWaitEvent(e->s_c, e->ev[2], 0));
        FVB_CUDA(cudaEventRecord(e->ev[3], e->s_c));
        if ((rc = fvb_plan_execute_ex(pl, batch_in_dev, batch_out_dev, nullptr, nullptr, 0, -1, 1, dt, h, gamma,
                                      with_reduction, e->d_lam, lam_patch_dev, e->s_c)))
            return rc;
        FVB_CUDA(cudaEventRecord(e->ev[4], e->s_c));
        FVB_CUDA(cudaStreamWaitEvent(e->s_s, e->ev[4], 0));
        for (int c = 0; c < chunks; ++c) {
            const long long lo = (long long)c * cp, hi = std::min((long long)T, lo + cp);
            if ((rc = scatter(lo, hi))) return rc;
            if (staged && c > 0 && (rc = host_scatter(lo - cp, lo, (c - 1) & 1))) return rc;
        }
        if (staged && (rc = host_scatter((long long)(chunks - 1) * cp, T, (chunks - 1) & 1))) return rc;
        steps_run = 1;
    } else {
        for (int c = 0; c < chunks; ++c) {
            const long long lo = (long long)c * cp, hi = std::min((long long)T, lo + cp);
            cudaEvent_t ev_g = e->ev[2 + 3 * c], ev_s = e->ev[3 + 3 * c], ev_c = e->ev[4 + 3 * c];
            if ((rc = gather(lo, hi))) return rc;
            FVB_CUDA(cudaEventRecord(ev_g, e->s_g));
            FVB_CUDA(cudaStreamWaitEvent(e->s_c, ev_g, 0));
            FVB_CUDA(cudaEventRecord(ev_s, e->s_c));
            if ((rc = fvb_plan_execute_ex(pl, batch_in_dev, batch_out_dev, nullptr, nullptr, lo, hi, 0, dt, h, gamma,
                                          with_reduction, e->d_lam + c, lam_patch_dev, e->s_c)))
                return rc;
            FVB_CUDA(cudaEventRecord(ev_c, e->s_c));
            FVB_CUDA(cudaStreamWaitEvent(e->s_s, ev_c, 0));
            if ((rc = scatter(lo, hi))) return rc;
            // host-staged: copy out the previous chunk while this one runs
            if (staged && c > 0 && (rc = host_scatter(lo - cp, lo, (c - 1) & 1))) return rc;
        }
        if (staged && (rc = host_scatter((long long)(chunks - 1) * cp, T, (chunks - 1) & 1))) return rc;
        steps_run = chunks;
    }
    if (reduce) {
        FVB_CUDA(cudaMemcpyAsync(e->h_lam, e->d_lam, sizeof(double) * chunks, cudaMemcpyDeviceToHost, e->s_c));
    }
    for (cudaStream_t s : {e->s_g, e->s_c, e->s_s}) {
        FVB_CUDA(cudaEventRecord(ev_end, s));
        FVB_CUDA(cudaStreamWaitEvent(st, ev_end, 0));
    }
    FVB_CUDA(cudaStreamSynchronize(st));
    // compute time: the step kernels' device intervals (step start -> step end per chunk)
    double compute = 0.0;
    for (int c = 0; c < steps_run; ++c) {
        float ms = 0.f;
        FVB_CUDA(cudaEventElapsedTime(&ms, e->ev[3 + 3 * c], e->ev[4 + 3 * c]));
        compute += ms * 1e-3;
    }
    if (compute_seconds_out) *compute_seconds_out = compute;
    if (reduced_out) {
        double r = 0.0;  // max(0, max of the chunk slots): exact
        if (reduce)
            for (int c = 0; c < chunks; ++c)
                if (e->h_lam[c] > r) r = e->h_lam[c];
        *reduced_out = r;
    }
    return FVB_OK;
}
