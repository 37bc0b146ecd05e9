// pencil.cu -- launcher of the fused 2D pencil kernel (fused2d.cuh) for one
// patch size.  Compiled once per P with -DFVB_P=<P> (build.py) so the
// instances build in parallel.
#include <cstdlib>

#include <cstdint>

#include "fused2d.cuh"
#include "fused2d_tile.cuh"
#include "fused2d_tma.cuh"
#include "host.h"

#ifndef FVB_P
#error "compile pencil.cu with -DFVB_P=<patch size>"
#endif

namespace fvb {
namespace {

template <class Eq, int P, int C, int R, int WARPS, int MINB, int RING, int LS = 1, bool V16 = false>
int launch_v(const StepArgs& a, cudaStream_t st) {
    auto kern = fused2d_pencil_kernel<Eq, P, C, WARPS, R, MINB, RING, LS, V16>;
    constexpr size_t smem = WARPS * pencil_smem_per_warp<P, C, RING, Eq::kUnknowns>();
    static PerDevice occ_dev;
    int& occ = occ_dev();
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

// The TMA-streamed kernel (fused2d_tma.cuh): SoA-ordered batches (patch
// stride <= unknown stride, 16-byte aligned), p | 32, >= 32/p patches.
// Returns 1 if the batch does not qualify (caller launches the cp.async kernel).
template <class Eq, int P, int R, int MINB, int RING, int RS = 2>
int launch_t(const StepArgs& a, cudaStream_t st) {
    if constexpr (32 % P != 0 || (P + 2) % RS != 0 || (P + 2) / RS < RING - 1) {
        return 1;
    } else {
        constexpr int G = 32 / P;
        const long long E = P + 2;
        if (a.in.l != 1 || a.in.p <= 0 || a.in.k <= 0 || a.in.p % 2 != 0 || a.in.k % 2 != 0 ||
            reinterpret_cast<std::uintptr_t>(a.q_in) % 16 != 0 || a.t1 - a.t0 < G ||
            a.t1 >= (1LL << 31) - (1LL << 24))
            return 1;
        // dimensions ordered by stride: SoA [col][row][patch][k], AoSoA [col][row][k][patch]
        const bool pm = a.in.k < a.in.p;
        constexpr int N = Eq::kUnknowns;
        const unsigned long long np = (unsigned long long)a.t1, nk = (unsigned long long)N;
        const unsigned long long sp = (unsigned long long)a.in.p * 8, sk = (unsigned long long)a.in.k * 8;
        const unsigned long long dims[4] = {(unsigned long long)E, (unsigned long long)E, pm ? nk : np,
                                            pm ? np : nk};
        const unsigned long long strides[3] = {(unsigned long long)E * 8, pm ? sk : sp, pm ? sp : sk};
        const unsigned g = G, n = N;
        const unsigned row_box[4] = {(unsigned)E, (unsigned)RS, pm ? n : g, pm ? g : n};
        const unsigned halo_box[4] = {2, (unsigned)P, pm ? n : g, pm ? g : n};
        CUtensorMap rows, halo;
        if (!tensor_map_4d(&rows, a.q_in, dims, strides, row_box) ||
            !tensor_map_4d(&halo, a.q_in, dims, strides, halo_box))
            return 1;
        auto kern = pm ? fused2d_pencil_tma_kernel<Eq, P, R, MINB, RING, RS, true>
                       : fused2d_pencil_tma_kernel<Eq, P, R, MINB, RING, RS, false>;
        constexpr size_t smem = pencil_tma_smem<P, RING, RS, N>();
        static PerDevice occ_dev[2];
        int& occ = occ_dev[pm]();
        if (occ == 0) {
            FVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32, smem);
            if (occ <= 0) occ = 1;
        }
        const long long groups = (a.t1 - a.t0 + G - 1) / G;
        long long blocks = groups;
        const long long cap = (long long)sm_count() * occ;
        if (blocks > cap) blocks = cap;
        kern<<<(unsigned)blocks, 32, smem, st>>>(a, rows, halo);
        return check_launch("fused2d_pencil_tma_kernel");
    }
}

int variant();

template <class Eq, int P, int R, int NB, int MINB, bool FUSE>
int tile_go_b(const StepArgs& a, cudaStream_t st) {
    constexpr size_t smem = tile_smem<P, Eq::kUnknowns, NB, FUSE>();
    auto kern = fused2d_tile_kernel<Eq, P, R, MINB, NB, FUSE>;
    static PerDevice occ_dev;
    int& occ = occ_dev();
    if (occ == 0) {
        FVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * P, smem);
        if (occ <= 0) occ = 1;
    }
    const long long groups = (a.t1 - a.t0 + tile::G - 1) / tile::G;
    long long blocks = groups;
    const long long cap = (long long)sm_count() * occ;
    if (blocks > cap) blocks = cap;
    kern<<<(unsigned)blocks, 32 * P, smem, st>>>(a);
    return check_launch("fused2d_tile_kernel");
}

template <class Eq, int P, int R, int NB, bool FUSE>
int tile_go(const StepArgs& a, cudaStream_t st) {
    // CTAs per SM: shared memory (NB groups staged per CTA), and >= 128
    // registers per thread (p = 3: 5 CTAs, 31.0 us, vs 6 CTAs at 96
    // registers with spills, 32.1 us -- FVB_TUNE_PENCIL_VARIANT = 3)
    constexpr size_t smem = tile_smem<P, Eq::kUnknowns, NB, FUSE>();
    constexpr int BY_SMEM = (int)((227u << 10) / smem);
    constexpr int BY_REGS = 65536 / (128 * 32 * P);
    constexpr int MINB = BY_SMEM < BY_REGS ? BY_SMEM : BY_REGS;
    if constexpr (BY_SMEM > MINB) {
        if (variant() == 3) return tile_go_b<Eq, P, R, NB, MINB + 1, FUSE>(a, st);
    }
    if constexpr (MINB > 1) {
        if (variant() == 7) return tile_go_b<Eq, P, R, NB, MINB - 1, FUSE>(a, st);
    }
    return tile_go_b<Eq, P, R, NB, MINB, FUSE>(a, st);
}

// The thread-per-patch kernel for tiny patches (fused2d_tile.cuh): SoA
// batches with exact strides whose per-unknown group segments are 16-byte
// aligned.  Returns 1 if the batch does not qualify.
template <class Eq, int P, int R>
int launch_tile(const StepArgs& a, cudaStream_t st) {
    if constexpr (P != 3) {  // p = 2 / 4: (p+2)^2 even -> conflicting 64-bit smem strides; pencils win
        return 1;
    } else {
        constexpr int N = Eq::kUnknowns;
        constexpr long long M = (P + 2) * (P + 2), Mi = P * P;
        const bool even = (M % 2 == 0) && (Mi % 2 == 0);
        if (a.in_tab != nullptr || a.layout != kLayoutSoA || a.in.l != 1 || a.out.l != 1 || a.in.p != M ||
            a.out.p != Mi || a.in.k != a.T * M || a.out.k != a.T * Mi ||
            reinterpret_cast<std::uintptr_t>(a.q_in) % 16 != 0 || reinterpret_cast<std::uintptr_t>(a.q_out) % 16 != 0 ||
            (a.T * M) % 2 != 0 || (a.T * Mi) % 2 != 0 || (!even && (a.t0 % 2 != 0 || a.t1 % 2 != 0)))
            return 1;
        // One staged group per CTA (the next one streams in once every warp
        // is done with the input).  FVB_TUNE_PENCIL_VARIANT = 2: two input
        // buffers, the next group streaming during the whole step -- measured
        // slower (C2: 34.7 vs 32.1 us; half the CTAs per SM).
        // FVB_TUNE_PENCIL_VARIANT = 4: each warp evaluates its row's AND its
        // column's cells (an interior cell's pressure twice, one barrier less)
        if (variant() == 2) return tile_go<Eq, P, R, 2, true>(a, st);
        if (variant() == 4) return tile_go<Eq, P, R, 1, false>(a, st);
        return tile_go<Eq, P, R, 1, true>(a, st);
    }
}

// Launch-shape variants (FVB_TUNE_PENCIL_VARIANT, tuning only).
int variant() { return tuning(FVB_TUNE_PENCIL_VARIANT); }

template <class Eq, int R>
int launch(const StepArgs& a, cudaStream_t st) {
    constexpr int P = FVB_P;
    constexpr int N = Eq::kUnknowns;
    // Measured on B200 (p=16, 2^20 patches): rows streamed by tensor-map TMA
    // copies, two haloed rows per copy, 3-slot ring (fused2d_tma.cuh) --
    // 3.50 ms cold / 73% of HBM sustained vs 4.00 ms / 66% for the cp.async
    // ring (the fallback, also for what the TMA path does not take: p not
    // dividing 32, AoS, unaligned or tiny batches).  cp.async shape: one
    // column per lane, 12 warps per SM (<= 170 registers, no spills) beats
    // two columns per lane (8 warps/SM or spills) and 16 warps/SM (128
    // registers: less ILP); one warp per CTA makes the group loop provably
    // warp-uniform (no BRA.DIV around shuffles / votes / syncwarps).
    if (a.layout == kLayoutAoS) {  // cells N apart; unknown pairs by 16-byte copies where aligned
        if constexpr (N % 2 == 0) {
            if (a.in_tab == nullptr && a.out_tab == nullptr && reinterpret_cast<std::uintptr_t>(a.q_in) % 16 == 0 &&
                reinterpret_cast<std::uintptr_t>(a.q_out) % 16 == 0 && a.in.p % 2 == 0 && a.out.p % 2 == 0 &&
                variant() != 9)
                return launch_v<Eq, P, 1, R, 1, 12, 3, N, true>(a, st);
        }
        return launch_v<Eq, P, 1, R, 1, 12, 3, N>(a, st);
    }
    // FVB_TUNE_PENCIL_VARIANT = 8 forces the cp.async ring (tests); the
    // measured-slower launch shapes of round 1 are no longer compiled.
    int rc = 1;
    // FVB_TUNE_PENCIL_VARIANT = 6 skips the thread-per-patch kernel (tests, A/B)
    if (variant() != 6 && variant() != 8) rc = launch_tile<Eq, P, R>(a, st);
    if (rc != 1) return rc;
    if (variant() != 8) rc = launch_t<Eq, P, R, 12, 3, 2>(a, st);
    if (rc != 1) return rc;
    return launch_v<Eq, P, 1, R, 1, 12, 3>(a, st);
}

}  // namespace

template <>
int pencil_launch<FVB_P>(const StepArgs& a, bool reduce, cudaStream_t st) {
    return with_physics<2>(a.physics, [&](auto tag) {
        using Eq = typename decltype(tag)::type;
        if (!reduce) return launch<Eq, kReduceNone>(a, st);
        // Measured on B200 (p=16, 2^20 patches, 100 steps under the power cap):
        // the filtered reduction is ~6% faster, so it is the default where
        // the physics has the lambda_below hook.
        // The p = 3 thread-per-patch kernel evaluates few cells per warp
        // between votes: exhaustive by default there (37.8 vs 38.7 us, C2).
        if constexpr (kHasLambdaBelow<Eq>) {
            const int f = tuning(FVB_TUNE_REDUCE_FILTER);
            if (a.lam_patch == nullptr && (f > 0 || (f < 0 && FVB_P != 3))) return launch<Eq, kReduceFiltered>(a, st);
        }
        return launch<Eq, kReduceAll>(a, st);
    });
}

}  // namespace fvb
