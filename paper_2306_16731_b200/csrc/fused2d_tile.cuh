// fused2d_tile.cuh -- the nested-parallel flavour for TINY 2D patches
// (p <= 4): a CTA of two warps owns 32 consecutive patches at a time, one
// patch per lane, the two warps split by AXIS.
//
// Why a different shape: with p = 3 a patch has 9 interior and 25 haloed
// cells, so the lane-per-column pencil (fused2d.cuh) spends most of its
// instructions on per-group overhead -- 5 rows per group through a ring,
// boundary faces recomputed in a separate phase, shuffles and an exchange
// row for every x-face (504 instructions per cell, 37% of the HBM roofline
// on C2).  A thread per patch has none of that (349 instructions per cell)
// but a whole patch is a long serial chain, and 32 staged patches per warp
// leave ~5 warps per SM: latency-bound (measured, ncu).  Splitting each
// patch between two warps halves the chain and, at the same shared memory
// per patch, doubles the warps:
//
//   * memory: per unknown, the CTA's 32 patches are ONE contiguous SoA
//     segment of 32 (p+2)^2 doubles (6.4 KB for p = 3); one thread moves the
//     N segments into shared memory with N bulk copies (cp.async.bulk,
//     completing on one mbarrier) and the N output segments back with bulk
//     stores (cp.async.bulk shared -> global).  The next group's copies are
//     issued as soon as both warps are done with the input.
//   * warp X (lane = patch): rows Y = 0..p-1, left to right: flux_x and the
//     x wave speed of every cell once, every x-face once, the x-update
//     Q + s*(G_l - G_r) of each interior cell into the output buffer.
//   * warp Y (lane = patch): columns, bottom to top: flux_y / wave speed of
//     every cell once, every y-face once, the face differences G_l - G_r of
//     each interior cell kept in registers; after a CTA barrier it finishes
//     every cell, acc_x + s*(G_l - G_r) -- the reference's update order and
//     association (microkernels.py:157-184), so the bits are unchanged.
//   * reduce: the two warps split the finished cells; filtered reduction,
//     fast path (XReal) + IEEE redo and the face algebra are fused2d.cuh's.
//   The pressure of an interior cell is evaluated by both warps (one per
//   axis): ~15 more FP64 operations per cell than a fused evaluation, bought
//   back many times by the parallelism.
//
// Conditions (host, pencil.cu): SoA with the exact batch strides, 16-byte
// aligned segments (T and the patch range even when (p+2)^2 or p^2 is odd).
// Everything else takes the pencil kernel.
// Reference realisation: run_patchwise (pkg/src/patchbench/executors.py:390-445).
#pragma once

#include "fused2d.cuh"
#include "fused3d.cuh"  // mbarrier / bulk-copy / named-barrier helpers

namespace fvb {

namespace tile {

constexpr int G = 32;  // patches per CTA group (one per lane)

template <int P, int N>
struct Geo {
    static constexpr int E = P + 2;
    static constexpr int M = E * E;   // haloed cells per patch
    static constexpr int Mi = P * P;  // interior cells per patch
    static constexpr int IN = G * M;  // doubles per unknown of a group's input
    static constexpr int OUT = G * Mi;
    static constexpr int HALF = (Mi + 1) / 2;  // reduce split: warp X cells [0, HALF), warp Y the rest
};

template <int P, int N>
struct alignas(128) CtaSmem {
    using Gm = Geo<P, N>;
    double in[N][Gm::IN];    // [k][patch][lin]
    double out[N][Gm::OUT];  // [k][patch][interior lin]: x-updated value, then the result
    double red[G];           // warp Y's per-patch maxima (lam_patch)
    unsigned long long mbar;
};

__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
                 "r"(slab::smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_shared() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

template <int P, int N>
struct Cells {
    const double* in;  // the lane's patch, [k * IN + lin]
    double* out;       // the lane's output slot, [k * OUT + interior lin]
    __device__ __forceinline__ void load(int x, int y, double (&q)[N]) const {  // x, y in [-1, P]
#pragma unroll
        for (int k = 0; k < N; ++k) q[k] = in[k * Geo<P, N>::IN + (x + 1) + Geo<P, N>::E * (y + 1)];
    }
};

// Warp X: the x-update of every interior cell into `out`.  s = dt/h, or
// 0.5*dt/h with R = XReal (doubled faces, fused2d.cuh face()).
template <class R, int P, class Eq, int N>
__device__ __forceinline__ void x_pass(const Eq& eq, const Cells<P, N>& c, double s, bool& bad) {
    using Gm = Geo<P, N>;
#pragma unroll 1
    for (int Y = 0; Y < P; ++Y) {
        double qL[N], fxL[N], lxL, gprev[N], d[N], dl;
        c.load(-1, Y, qL);
        pencil::eval<R, true, false>(eq, qL, fxL, lxL, d, dl, bad);
#pragma unroll
        for (int x = 0; x <= P; ++x) {
            double qR[N], fxR[N], lxR, g[N];
            c.load(x, Y, qR);
            pencil::eval<R, true, false>(eq, qR, fxR, lxR, d, dl, bad);
            pencil::face<R>(qL, qR, fxL, fxR, lxL, lxR, g);  // x-face at x - 1/2
            if (x > 0) {
                double acc[N];
#pragma unroll
                for (int k = 0; k < N; ++k) acc[k] = qL[k];
                rusanov_update(acc, gprev, g, s);
#pragma unroll
                for (int k = 0; k < N; ++k) c.out[k * Gm::OUT + (x - 1) + P * Y] = acc[k];
            }
#pragma unroll
            for (int k = 0; k < N; ++k) gprev[k] = g[k], qL[k] = qR[k], fxL[k] = fxR[k];
            lxL = lxR;
        }
    }
}

// Warp Y: the y-face differences G_{y-1/2} - G_{y+1/2} of every interior cell.
template <class R, int P, class Eq, int N>
__device__ __forceinline__ void y_pass(const Eq& eq, const Cells<P, N>& c, double (&t)[P][P][N], bool& bad) {
#pragma unroll
    for (int x = 0; x < P; ++x) {
        double qD[N], fyD[N], lyD, gprev[N], d[N], dl;
        c.load(x, -1, qD);
        pencil::eval<R, false, true>(eq, qD, d, dl, fyD, lyD, bad);
#pragma unroll
        for (int y = 0; y <= P; ++y) {
            double qU[N], fyU[N], lyU, g[N];
            c.load(x, y, qU);
            pencil::eval<R, false, true>(eq, qU, d, dl, fyU, lyU, bad);
            pencil::face<R>(qD, qU, fyD, fyU, lyD, lyU, g);  // y-face at y - 1/2
            if (y > 0) {
#pragma unroll
                for (int k = 0; k < N; ++k) t[y - 1][x][k] = gprev[k] - g[k];
            }
#pragma unroll
            for (int k = 0; k < N; ++k) gprev[k] = g[k], qD[k] = qU[k], fyD[k] = fyU[k];
            lyD = lyU;
        }
    }
}

// max_n lambda_n of a finished cell: the fast path where the policy
// certifies the state, else IEEE double (a per-cell fallback: the results
// are already final, only this evaluation needs the slow path).
template <class Eq, int N>
__device__ __forceinline__ double lambda_of(const Eq& eq, const double (&q)[N]) {
    if constexpr (kHasFastPath<Eq>) {
        bool bad = false;
        const double v = pencil::cell_lambda<XReal>(eq, q, bad);
        if (!bad) return v;
    }
    bool unused = false;
    return pencil::cell_lambda<double>(eq, q, unused);
}

}  // namespace tile

template <int P, int N>
constexpr size_t tile_smem() {
    return sizeof(tile::CtaSmem<P, N>);
}

// CTA = warp X + warp Y; group g (32 patches from t0 + 32 g) for
// g = blockIdx.x, + gridDim.x, ...  The host guarantees 16-byte aligned segments.
template <class Eq, int P, int RED, int MINB>
__global__ void __launch_bounds__(64, MINB) fused2d_tile_kernel(StepArgs a) {
    using namespace tile;
    constexpr int N = Eq::kUnknowns;
    using Gm = Geo<P, N>;
    static_assert(Eq::kDim == 2, "2D patches");
    static_assert(RED != kReduceFiltered || kHasLambdaBelow<Eq>, "filtered reduction needs lambda_below");
    const Eq eq(a.gamma);

    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto& S = *reinterpret_cast<CtaSmem<P, N>*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31;
    const bool wx = tid < 32;  // warp X (else warp Y); warp-uniform
    const long long t0 = a.t0, t1 = a.t1;
    const long long groups = (t1 - t0 + G - 1) / G;
    const double scale = step_scale(a);
    const bool fast = step_fast(a, scale);

    auto issue_load = [&](long long g) {  // thread 0: the group's N input segments
        const long long first = t0 + g * G;
        const unsigned bytes = (unsigned)(min((long long)G, t1 - first) * Gm::M * 8);
        slab::mbar_expect_tx(&S.mbar, N * bytes);
#pragma unroll
        for (int k = 0; k < N; ++k) slab::bulk_g2s(&S.in[k][0], a.q_in + k * a.in.k + first * Gm::M, bytes, &S.mbar);
    };

    if (tid == 0) {
        slab::mbar_init(&S.mbar, 1);
        slab::fence_mbar_init();
    }
    __syncthreads();
    long long g = blockIdx.x;
    if (tid == 0 && g < groups) issue_load(g);

    double red = 0.0;
    LamFilter lf;
    lf.init();
    unsigned phase = 0;
    for (; g < groups; g += gridDim.x) {
        const long long first = t0 + g * G;
        const int np = (int)min((long long)G, t1 - first);
        const bool valid = lane < np;
        const long long patch = first + (valid ? lane : 0);  // stand-in input for a partial group's tail
        double s = scale;
        bool lane_fast = fast;
        if (a.dt_patch != nullptr) {  // local time stepping: this lane's patch's dt
            s = patch_scale(a, scale, patch);
            lane_fast = step_fast(a, s);
        }
        const Cells<P, N> c{&S.in[0][(valid ? lane : 0) * Gm::M], &S.out[0][lane * Gm::Mi]};
        if (tid == 0) bulk_wait_read();  // the previous group's stores have read `out`
        __syncthreads();
        slab::mbar_wait(&S.mbar, phase);
        phase ^= 1u;

        // ---- the two axis passes (fast path, IEEE redo if any state is uncertified)
        double t[P][P][N];
        bool fold = false;
        if constexpr (kHasFastPath<Eq>) {
            bool bad = !lane_fast;
            if (wx) x_pass<XReal>(eq, c, 0.5 * s, bad);
            else y_pass<XReal>(eq, c, t, bad);
            fold = !slab::slot_any(1, 64, bad && valid);  // also the barrier after the passes
        } else {
            __syncthreads();
        }
        if (!fold) {
            bool unused = false;
            if (wx) x_pass<double>(eq, c, s, unused);
            else y_pass<double>(eq, c, t, unused);
            __syncthreads();
        }
        if (tid == 0 && g + gridDim.x < groups) issue_load(g + gridDim.x);  // `in` is free
        if (!wx) {  // warp Y finishes every cell: acc_x + s * (G_l - G_r)
            const double sf = fold ? 0.5 * s : s;
#pragma unroll
            for (int y = 0; y < P; ++y)
#pragma unroll
                for (int x = 0; x < P; ++x)
#pragma unroll
                    for (int k = 0; k < N; ++k) {
                        double& o = c.out[k * Gm::OUT + x + P * y];
                        o = o + sf * t[y][x][k];
                    }
        }
        __syncthreads();
        if (tid == 0) {
            fence_async_shared();  // generic writes of `out` -> the bulk stores
            const unsigned bytes = (unsigned)(np * Gm::Mi * 8);
#pragma unroll
            for (int k = 0; k < N; ++k) bulk_s2g(a.q_out + k * a.out.k + first * Gm::Mi, &S.out[k][0], bytes);
            bulk_commit();
        }

        // ---- reduce: warp X cells [0, HALF), warp Y [HALF, Mi)
        double pred = 0.0;
        if constexpr (RED != kReduceNone) {
            constexpr int H = Gm::HALF;
            const int c0 = wx ? 0 : H, nc = wx ? H : Gm::Mi - H;
            if constexpr (RED == kReduceAll) {
#pragma unroll 1
                for (int i = 0; i < nc; ++i) {
                    double q[N];
#pragma unroll
                    for (int k = 0; k < N; ++k) q[k] = c.out[k * Gm::OUT + c0 + i];
                    running_max(pred, lambda_of(eq, q));
                }
            } else {  // filtered: only cells the policy cannot place under tau
                unsigned need = 0;
#pragma unroll 1
                for (int i = 0; i < nc; ++i) {
                    double q[N];
#pragma unroll
                    for (int k = 0; k < N; ++k) q[k] = c.out[k * Gm::OUT + c0 + i];
                    if (valid && !eq.lambda_below(q, lf.tau_lo)) need |= 1u << i;
                }
                if (__any_sync(0xffffffffu, need != 0)) {
#pragma unroll 1
                    for (int i = 0; i < nc; ++i) {
                        if (!(need >> i & 1u)) continue;
                        double q[N];
#pragma unroll
                        for (int k = 0; k < N; ++k) q[k] = c.out[k * Gm::OUT + c0 + i];
                        running_max(pred, lambda_of(eq, q));
                    }
                    lf.raise(pred);
                }
            }
            if (!valid) pred = 0.0;
            running_max(red, pred);
            if (RED == kReduceAll && a.lam_patch != nullptr) {  // the patch's max over both warps
                if (!wx) S.red[lane] = pred;
                __syncthreads();
                if (wx && valid) {
                    double v = pred;
                    running_max(v, S.red[lane]);
                    a.lam_patch[patch] = v;
                }
            }
        }
    }
    if (tid == 0) bulk_wait_all();
    if (RED != kReduceNone && a.lam_bits != nullptr) {
        red = warp_max(red);
        if (lane == 0) atomic_max_nonneg(a.lam_bits, red);
    }
}

}  // namespace fvb
