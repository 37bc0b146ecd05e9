// slab3d.cu -- launcher of the fused 3D plane-walk kernel (fused3d.cuh) for
// one patch size.  Compiled once per P with -DFVB_P3=<P> (build.py).
#include <cstdint>
#include <cstdlib>

#include "fused3d.cuh"
#include "fused3d_warp.cuh"
#include "host.h"

#ifndef FVB_P3
#error "compile slab3d.cu with -DFVB_P3=<patch size>"
#endif

namespace fvb {
namespace {

template <class Eq, int P, int R, int SLOTS, int RING, int MINB, int LS = 1>
int launch_v(const StepArgs& a, cudaStream_t st) {
    auto kern = fused3d_slab_kernel<Eq, P, SLOTS, RING, R, MINB, LS>;
    constexpr int threads = SLOTS * slab::Geo3<P>::TH;
    constexpr size_t smem = SLOTS * slab_smem_per_slot<P, RING, Eq::kUnknowns>();
    static PerDevice occ_dev;
    int& occ = occ_dev();
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

// two-warp-slot kernel: CTAs per SM for ~12 resident warps (<= ~170 registers)
template <int P>
constexpr int kSlotMinBlocks = (384 / (slab::Geo3<P>::TH < 32 ? 32 : slab::Geo3<P>::TH)) > 0
                                    ? (384 / (slab::Geo3<P>::TH < 32 ? 32 : slab::Geo3<P>::TH))
                                    : 1;
// slots per CTA: one for slots of whole warps, a warp's worth of sub-warp
// slots (p = 2: 4 patches, p = 3 / 4: 2 patches per warp)
template <int P>
constexpr int kSlots = slab::Geo3<P>::TH < 32 ? 32 / slab::Geo3<P>::TH : 1;

// The 4-D tensor map of the haloed input batch the one-warp kernel streams
// its z-planes through: [lin][plane][patch][k] or [lin][plane][k][patch]
// (dimensions ordered by stride), box = one plane of every unknown.  False
// if the batch does not fit TMA's rules (16-byte aligned base and strides,
// cell stride 1, < 2^31 - 2^24 patches) or the driver lacks the encoder.
bool plane_map(CUtensorMap* tm, int* patch_d2, const StepArgs& a, int P, int N) {
    const long long M2 = (long long)(P + 2) * (P + 2);
    if (a.in_tab != nullptr || a.q_in == nullptr) return false;  // per-patch arrays (SHARED mode): no one tensor
    if (a.layout == kLayoutAoS) {  // a plane is N*M2 interleaved doubles: [M2][N][plane][patch], box {M2, N, 1, 1}
        if (a.in.l != N || a.in.k != 1 || a.in.p <= 0 || a.in.p % 2 != 0 ||
            reinterpret_cast<std::uintptr_t>(a.q_in) % 16 != 0 || a.t1 >= (1LL << 31) - (1LL << 24) ||
            (M2 * 8) % 16 != 0 || M2 > 256)
            return false;
        const unsigned long long dims[4] = {(unsigned long long)M2, (unsigned long long)N,
                                            (unsigned long long)(P + 2), (unsigned long long)a.t1};
        const unsigned long long strides[3] = {(unsigned long long)M2 * 8, (unsigned long long)(N * M2) * 8,
                                               (unsigned long long)a.in.p * 8};
        const unsigned box[4] = {(unsigned)M2, (unsigned)N, 1, 1};
        *patch_d2 = 0;
        return tensor_map_4d(tm, a.q_in, dims, strides, box);
    }
    if (a.in.l != 1 || a.in.k <= 0 || a.in.p <= 0 || a.in.k % 2 != 0 || a.in.p % 2 != 0 ||
        reinterpret_cast<std::uintptr_t>(a.q_in) % 16 != 0 || a.t1 >= (1LL << 31) - (1LL << 24) ||
        (M2 * 8) % 16 != 0)
        return false;
    const bool d2 = a.in.p <= a.in.k;  // SoA: patches inside an unknown's block
    const unsigned long long np = (unsigned long long)a.t1, nk = (unsigned long long)N;
    const unsigned long long sp = (unsigned long long)a.in.p * 8, sk = (unsigned long long)a.in.k * 8;
    const unsigned long long dims[4] = {(unsigned long long)M2, (unsigned long long)(P + 2), d2 ? np : nk,
                                        d2 ? nk : np};
    const unsigned long long strides[3] = {(unsigned long long)M2 * 8, d2 ? sp : sk, d2 ? sk : sp};
    const unsigned box[4] = {(unsigned)M2, 1, d2 ? 1u : (unsigned)nk, d2 ? (unsigned)nk : 1u};
    *patch_d2 = d2 ? 1 : 0;
    return tensor_map_4d(tm, a.q_in, dims, strides, box);
}

// One warp per patch (fused3d_warp.cuh, p = 8 only); the slot kernel where
// the batch cannot be described by a plane map.
template <class Eq, int P, int R, int RING, int MINB, int LS = 1>
int launch_w(const StepArgs& a, cudaStream_t st) {
    CUtensorMap tm;
    int patch_d2 = 0;
    if constexpr (P != 8) {
        return launch_v<Eq, P, R, kSlots<P>, 4, 6, LS>(a, st);
    } else if (!plane_map(&tm, &patch_d2, a, P, Eq::kUnknowns)) {
        return launch_v<Eq, P, R, kSlots<P>, 4, kSlotMinBlocks<P>, LS>(a, st);
    } else {
        auto kern = fused3d_warp_kernel<Eq, P, RING, R, MINB, LS>;
        constexpr size_t smem = sizeof(slabw::WarpSmem<P, RING, Eq::kUnknowns>);
        static PerDevice occ_dev;
        int& occ = occ_dev();
        if (occ == 0) {
            FVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32, smem);
            if (occ <= 0) occ = 1;
        }
        long long blocks = a.t1 - a.t0;
        const long long cap = (long long)sm_count() * occ;
        if (blocks > cap) blocks = cap;
        kern<<<(unsigned)blocks, 32, smem, st>>>(a, tm, patch_d2);
        return check_launch("fused3d_warp_kernel");
    }
}

int variant() { return tuning(FVB_TUNE_SLAB_VARIANT); }

// Default launch for p = 8 (SoA / AoSoA): one warp per patch, 2-plane ring,
// 8 CTAs per SM (251 registers; the ring depth does not matter, the 8th
// warp does).  Other p and AoS: the two-warp slot kernel.
template <int P>
constexpr bool kWarpDefault = (P == 8);

template <class Eq, int R>
int launch(const StepArgs& a, cudaStream_t st) {
    constexpr int P = FVB_P3;
    constexpr int N = Eq::kUnknowns;
    if (a.layout == kLayoutAoS) {  // cells N apart
        if constexpr (kWarpDefault<P>) {
            if (variant() != 5) return launch_w<Eq, P, R, 2, 8, N>(a, st);
        }
        return launch_v<Eq, P, R, kSlots<P>, 4, kSlotMinBlocks<P>, N>(a, st);
    }
    // FVB_TUNE_SLAB_VARIANT = 5 forces the two-warp slot kernel for p = 8
    // (tests); the measured-slower launch shapes of round 1 are no longer compiled.
    if (variant() == 5) return launch_v<Eq, P, R, kSlots<P>, 4, kSlotMinBlocks<P>>(a, st);
    if constexpr (kWarpDefault<P>) return launch_w<Eq, P, R, 2, 8>(a, st);
    return launch_v<Eq, P, R, kSlots<P>, 4, kSlotMinBlocks<P>>(a, st);
}

template <class Eq>
int launch_physics(const StepArgs& a, bool reduce, cudaStream_t st) {
    if (!reduce) return launch<Eq, kReduceNone>(a, st);
    // The filtered reduction (no per-patch maxima) pays in the one-warp
    // kernel (p = 8: -7% instructions, -4% time, ncu) but costs 5% in the
    // two-warp slot kernel, whose vote-guarded branch loses the uniform
    // datapath; FVB_TUNE_REDUCE_FILTER = 0 / 1 overrides.  Only physics with
    // the lambda_below hook can filter.
    if constexpr (kHasLambdaBelow<Eq>) {
        const int f = tuning(FVB_TUNE_REDUCE_FILTER);
        const bool warp_kernel = kWarpDefault<FVB_P3> && variant() == 0;
        if (a.lam_patch == nullptr && (f == 1 || (f < 0 && warp_kernel))) return launch<Eq, kReduceFiltered>(a, st);
    }
    return launch<Eq, kReduceAll>(a, st);
}

}  // namespace

template <>
int slab_launch<FVB_P3>(const StepArgs& a, bool reduce, cudaStream_t st) {
    return with_physics<3>(a.physics, [&](auto tag) { return launch_physics<typename decltype(tag)::type>(a, reduce, st); });
}

}  // namespace fvb
