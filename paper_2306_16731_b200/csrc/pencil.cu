// pencil.cu -- launcher of the fused 2D pencil kernel (fused2d.cuh) for one
// patch size.  Compiled once per P with -DFVB_P=<P> (build.py) so the
// instances build in parallel.
#include <cstdlib>

#include "fused2d.cuh"
#include "host.h"

#ifndef FVB_P
#error "compile pencil.cu with -DFVB_P=<patch size>"
#endif

namespace fvb {
namespace {

template <int P, int C, int R, int WARPS, int MINB, int RING, int LS = 1>
int launch_v(const StepArgs& a, cudaStream_t st) {
    auto kern = fused2d_pencil_kernel<P, C, WARPS, R, MINB, RING, LS>;
    constexpr size_t smem = WARPS * pencil_smem_per_warp<P, C, RING>();
    static int occ = 0;
    if (occ == 0) {
        FVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, WARPS * 32, smem);
        if (occ <= 0) occ = 1;
    }
    constexpr int G = pencil::Geo<P, C>::G;
    const long long groups = (a.t1 - a.t0 + G - 1) / G;
    long long blocks = (groups + WARPS - 1) / WARPS;
    const long long cap = (long long)sm_count() * occ;
    if (blocks > cap) blocks = cap;
    kern<<<(unsigned)blocks, WARPS * 32, smem, st>>>(a);
    return check_launch("fused2d_pencil_kernel");
}

// Launch-shape variants (FVB_TUNE_PENCIL_VARIANT, tuning only).
int variant() { return tuning(FVB_TUNE_PENCIL_VARIANT); }

template <int R>
int launch(const StepArgs& a, cudaStream_t st) {
    constexpr int P = FVB_P;
    // Measured on B200 (p=16, 2^20 patches): one column per lane, 12 warps per
    // SM (<= 170 registers, no spills) beats two columns per lane (8 warps/SM
    // or spills) and 16 warps/SM (128 registers: less ILP).  One warp per CTA
    // makes the group loop provably warp-uniform: no divergence checks
    // (BRA.DIV) around the shuffles / votes / syncwarps, 5% fewer
    // instructions, 1.2% faster (variant 4: the same at 4 warps per CTA).
    if (a.layout == kLayoutAoS) return launch_v<P, 1, R, 1, 12, 3, 4>(a, st);  // cells N = 4 apart
#if FVB_P == 16
    switch (variant()) {
        case 1: return launch_v<P, 1, R, 4, 3, 4>(a, st);
        case 2: return launch_v<P, 2, R, 4, 2, 4>(a, st);
        case 3: return launch_v<P, 1, R, 4, 4, 3>(a, st);
        case 4: return launch_v<P, 1, R, 4, 3, 3>(a, st);
        case 5: return launch_v<P, 1, R, 1, 12, 4>(a, st);
        default: break;
    }
#endif
    return launch_v<P, 1, R, 1, 12, 3>(a, st);
}

}  // namespace

template <>
int pencil_launch<FVB_P>(const StepArgs& a, bool reduce, cudaStream_t st) {
    if (!reduce) return launch<kReduceNone>(a, st);
    // Measured on B200 (p=16, 2^20 patches, 100 steps under the power cap):
    // the filtered reduction is ~6% faster, so it is the default.
    const bool filtered = tuning(FVB_TUNE_REDUCE_FILTER) != 0;
    return (a.lam_patch == nullptr && filtered) ? launch<kReduceFiltered>(a, st)
                                                : launch<kReduceAll>(a, st);
}

}  // namespace fvb
