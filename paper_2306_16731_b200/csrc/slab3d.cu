// slab3d.cu -- launcher of the fused 3D plane-walk kernel (fused3d.cuh) for
// one patch size.  Compiled once per P with -DFVB_P3=<P> (build.py).
#include <cstdlib>

#include "fused3d.cuh"
#include "host.h"

#ifndef FVB_P3
#error "compile slab3d.cu with -DFVB_P3=<patch size>"
#endif

namespace fvb {
namespace {

template <int P, int R, int SLOTS, int RING, int MINB, int LS = 1>
int launch_v(const StepArgs& a, cudaStream_t st) {
    auto kern = fused3d_slab_kernel<P, SLOTS, RING, R, MINB, LS>;
    constexpr int threads = SLOTS * slab::Geo3<P>::TH;
    constexpr size_t smem = SLOTS * slab_smem_per_slot<P, RING>();
    static int occ = 0;
    if (occ == 0) {
        FVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (occ <= 0) occ = 1;
    }
    const long long patches = a.t1 - a.t0;
    long long blocks = (patches + SLOTS - 1) / SLOTS;
    const long long cap = (long long)sm_count() * occ;
    if (blocks > cap) blocks = cap;
    kern<<<(unsigned)blocks, threads, smem, st>>>(a);
    return check_launch("fused3d_slab_kernel");
}

int variant() { return tuning(FVB_TUNE_SLAB_VARIANT); }

template <int R>
int launch(const StepArgs& a, cudaStream_t st) {
    constexpr int P = FVB_P3;
    if (a.layout == kLayoutAoS) return launch_v<P, R, 1, 4, 6, 5>(a, st);  // cells N = 5 apart
    switch (variant()) {
        case 1: return launch_v<P, R, 1, 3, 7>(a, st);
        case 2: return launch_v<P, R, 2, 3, 3>(a, st);
        case 3: return launch_v<P, R, 1, 3, 6>(a, st);
        case 4: return launch_v<P, R, 1, 2, 8>(a, st);
        default: break;
    }
    return launch_v<P, R, 1, 4, 6>(a, st);
}

}  // namespace

template <>
int slab_launch<FVB_P3>(const StepArgs& a, bool reduce, cudaStream_t st) {
    if (!reduce) return launch<kReduceNone>(a, st);
    // Measured on B200 (3D p=8, 100k patches): the filtered reduction is ~5%
    // slower here (its vote sits on the barrier-bound critical path of the
    // plane walk), so the exhaustive reduction is the default;
    // FVB_TUNE_REDUCE_FILTER=1 selects the filter.
    const bool filtered = tuning(FVB_TUNE_REDUCE_FILTER) == 1;
    return (a.lam_patch == nullptr && filtered) ? launch<kReduceFiltered>(a, st)
                                                : launch<kReduceAll>(a, st);
}

}  // namespace fvb
