// host.h -- internal host-side interface between the translation units of
// libfvb.so (not part of the C ABI; include/fvb.h is).
//
//   fvb.cu      C ABI: validation, errors, plans, graphs, step dispatch
//   pencil.cu   fused 2D pencil kernel, compiled once per patch size P
//   slab3d.cu   fused 3D plane-walk kernel (TMA-streamed z-planes), one per P
//   generic.cu  fused shared-memory kernel (odd / large 3D, large 2D patches)
//   cascade.cu  per-step kernels of the cascade / graph flavours
//   misc.cu     seeded field, AoS<->SoA, microkernel probe, admissibility
#pragma once

#include <cuda.h>  // CUtensorMap
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <thread>

#include "../../include/fvb.h"
#include "common.cuh"
#include "physics.cuh"

#define FVB_CUDA(call)                                                                       \
    do {                                                                                      \
        cudaError_t _e = (call);                                                              \
        if (_e != cudaSuccess)                                                                \
            return ::fvb::fail(FVB_ECUDA, "%s failed: %s (%s:%d)", #call,                     \
                               cudaGetErrorString(_e), __FILE__, __LINE__);                   \
    } while (0)

namespace fvb {

// errors / device facts (fvb.cu)
int fail(int code, const char* fmt, ...);
int check_launch(const char* what);
long long ipow_h(long long b, int e);
int validate_shape(int dim, int p, int64_t T);
int sm_count();

// Host-side caches keyed by the caller's stream (reduction slots, cached
// plans and their scratch, transfer engines): cudaStreamPerThread is ONE
// handle for one stream per host thread, whose work may overlap, so for it
// the key includes the calling thread.
// Scope in which this thread's calls use the relaxed stream-capture mode:
// a step first reached inside a user's CUDA-graph capture may allocate its
// plan's scratch or instantiate its task graph (eager, not captured) while
// its kernels are captured.
struct RelaxedCapture {
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&mode); }
    ~RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&mode); }
    RelaxedCapture(const RelaxedCapture&) = delete;
    RelaxedCapture& operator=(const RelaxedCapture&) = delete;
};

inline size_t stream_thread_key(const void* stream) {
    return stream == reinterpret_cast<const void*>(cudaStreamPerThread)
               ? std::hash<std::thread::id>{}(std::this_thread::get_id())
               : 0;
}
int smem_optin();
long long blocks_for(long long work, int threads, int per_sm);
bool tensor_map_4d(CUtensorMap* tm, const void* base, const unsigned long long dims[4],
                   const unsigned long long strides_bytes[3], const unsigned box[4]);

// One value per device ordinal: once-only launch setup (the shared-memory
// opt-in attribute, occupancy) is per device context, and one process may
// drive several GPUs.
struct PerDevice {
    int v[64] = {};
    int& operator()() {
        int d = 0;
        cudaGetDevice(&d);
        return v[d & 63];
    }
};

// launch tuning (fvb_set_tuning, fvb.cu)
int tuning(int key);

// physics policies (physics.cuh): with_physics<D>(id, f) calls f(Tag<Eq>{})
// for the policy FVB_PHYSICS_* `id` of dimension D.  The host batch format
// is the reference's BatchShape (N = d + 2 unknowns, patchdata.py:93-99), so
// every policy compiled in carries d + 2 unknowns.
int physics();  // the process-wide selection (fvb_set_physics, fvb.cu)
template <class T>
struct Tag {
    using type = T;
};
template <int D, class F>
auto with_physics(int id, F&& f) {
    static_assert(Euler<D>::kUnknowns == D + 2 && EulerPlain<D>::kUnknowns == D + 2, "BatchShape has d+2 unknowns");
    if (id == FVB_PHYSICS_EULER_PLAIN) return f(Tag<EulerPlain<D>>{});
    return f(Tag<Euler<D>>{});
}

// fused flavour
template <int P>
int pencil_launch(const StepArgs& a, bool reduce, cudaStream_t st);  // pencil.cu, one per P
#define FVB_PENCIL_SIZES(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) \
    X(14) X(15) X(16) X(32)
#define FVB_DECLARE_PENCIL(P) template <> int pencil_launch<P>(const StepArgs&, bool, cudaStream_t);
FVB_PENCIL_SIZES(FVB_DECLARE_PENCIL)
#undef FVB_DECLARE_PENCIL
template <int P>
int slab_launch(const StepArgs& a, bool reduce, cudaStream_t st);  // slab3d.cu, one per P
#define FVB_SLAB_SIZES(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)
#define FVB_DECLARE_SLAB(P) template <> int slab_launch<P>(const StepArgs&, bool, cudaStream_t);
FVB_SLAB_SIZES(FVB_DECLARE_SLAB)
#undef FVB_DECLARE_SLAB
long long generic_smem_bytes(int dim, int p);                              // generic.cu
int launch_generic(int dim, const StepArgs& a, bool reduce, cudaStream_t st);

// cascade / graph flavours (cascade.cu)
constexpr int kEltThreads = 256;
constexpr int kReduceThreads = 256;
struct CascadeFns {
    void *copy, *flux, *lam, *acc, *reduce;
};
CascadeFns cascade_fns(int dim, int physics);
int launch_cascade(int dim, const CascadeArgs& ca, bool reduce, cudaStream_t st);

}  // namespace fvb
