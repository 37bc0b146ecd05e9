// fused2d_tile.cuh -- the nested-parallel flavour for TINY 2D patches
// (p <= 4): a CTA of p warps owns 32 consecutive patches at a time, one
// patch per lane; warp r owns ROW r and COLUMN r of every patch.
//
// Why a different shape: with p = 3 a patch has 9 interior and 25 haloed
// cells, so the lane-per-column pencil (fused2d.cuh) spends most of its
// instructions on per-group overhead -- 5 rows per group through a ring,
// boundary faces recomputed in a separate phase, shuffles and an exchange
// row for every x-face (504 instructions per cell, 37% of the HBM roofline
// on C2).  A thread per patch has none of that (349 instructions per cell)
// but a whole patch is a long serial chain, and 32 staged patches per warp
// leave ~5 warps per SM: latency-bound (measured, ncu).  Splitting every
// patch between p warps cuts the chain to one row + one column and, at the
// same shared memory per patch, multiplies the warps by p:
//
//   * memory: per unknown, the CTA's 32 patches are ONE contiguous SoA
//     segment of 32 (p+2)^2 doubles (6.4 KB for p = 3); one thread moves the
//     N segments into shared memory with N bulk copies (cp.async.bulk,
//     completing on one mbarrier) and the N output segments back with bulk
//     stores (cp.async.bulk shared -> global).  The next group's copies are
//     issued as soon as every warp is done with the input.
//   * phase 1, warp r, row r: the microkernels of its cells once -- both
//     axes for its p interior cells (the y-flux / y wave speed published to
//     shared memory for their column), the x-axis for its two x-halo cells,
//     the y-axis for column r's two y-halo cells; its p+1 x-faces once and
//     the x-updates Q + s*(G_l - G_r) of its interior cells (registers);
//   * phase 2 (after a CTA barrier), warp r, column r: its p+1 y-faces from
//     the published fluxes, the differences G_l - G_r written over them;
//   * phase 3 (after a CTA barrier), warp r finishes row r: acc_x +
//     s*(G_l - G_r), the reference's update order and association
//     (microkernels.py:157-184), then the eigenvalues of its finished cells.
//   Face algebra, fast path (XReal) + IEEE redo and the filtered reduction
//   are fused2d.cuh's, so the bits are the reference's.  (The variant with
//   each warp evaluating its row's AND its column's cells -- an interior
//   cell's pressure twice, one barrier less -- is FVB_TUNE_PENCIL_VARIANT=4.)
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
};

template <int P, int N, int NB, bool FUSE = false>
struct alignas(128) CtaSmem {
    using Gm = Geo<P, N>;
    double in[NB][N][Gm::IN];  // [buffer][k][patch][lin]: NB = 2 streams the next group during this one
    // [k][patch][interior lin]: FUSE: the y-flux (k < N) and y wave speed
    // (k = N) of every interior cell, then the y-face differences, then the
    // result; else the y-face differences, then the result
    double out[N + (FUSE ? 1 : 0)][Gm::OUT];
    double red[P][G];          // per-row maxima of each patch (lam_patch)
    unsigned long long mbar[NB];
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
    __device__ __forceinline__ double& at(int k, int x, int y) const { return out[k * Geo<P, N>::OUT + x + P * y]; }
};

// Row r along x: flux_x / x wave speed of its p+2 cells, its p+1 x-faces,
// and the x-updates Q + s*(G_l - G_r) of its p interior cells (returned in
// acc).  s = dt/h, or 0.5*dt/h with R = XReal (doubled faces, fused2d.cuh face()).
template <class R, int P, class Eq, int N>
__device__ __forceinline__ void x_row(const Eq& eq, const Cells<P, N>& c, int r, double s, double (&acc)[P][N],
                                      bool& bad) {
    double qL[N], fxL[N], lxL, gprev[N], d[N], dl;
    c.load(-1, r, qL);
    pencil::eval<R, true, false>(eq, qL, fxL, lxL, d, dl, bad);
#pragma unroll
    for (int x = 0; x <= P; ++x) {
        double qR[N], fxR[N], lxR, g[N];
        c.load(x, r, qR);
        pencil::eval<R, true, false>(eq, qR, fxR, lxR, d, dl, bad);
        pencil::face<R>(qL, qR, fxL, fxR, lxL, lxR, g);  // x-face at x - 1/2
        if (x > 0) {
#pragma unroll
            for (int k = 0; k < N; ++k) acc[x - 1][k] = qL[k];
            rusanov_update(acc[x - 1], gprev, g, s);
        }
#pragma unroll
        for (int k = 0; k < N; ++k) gprev[k] = g[k], qL[k] = qR[k], fxL[k] = fxR[k];
        lxL = lxR;
    }
}

// Column r along y: flux_y / y wave speed of its p+2 cells, its p+1
// y-faces, and the face differences G_{y-1/2} - G_{y+1/2} of its p
// interior cells, parked in the output buffer for their row's warp.
template <class R, int P, class Eq, int N>
__device__ __forceinline__ void y_col(const Eq& eq, const Cells<P, N>& c, int r, bool& bad) {
    double qD[N], fyD[N], lyD, gprev[N], d[N], dl;
    c.load(r, -1, qD);
    pencil::eval<R, false, true>(eq, qD, d, dl, fyD, lyD, bad);
#pragma unroll
    for (int y = 0; y <= P; ++y) {
        double qU[N], fyU[N], lyU, g[N];
        c.load(r, y, qU);
        pencil::eval<R, false, true>(eq, qU, d, dl, fyU, lyU, bad);
        pencil::face<R>(qD, qU, fyD, fyU, lyD, lyU, g);  // y-face at y - 1/2
        if (y > 0) {
#pragma unroll
            for (int k = 0; k < N; ++k) c.at(k, r, y - 1) = gprev[k] - g[k];
        }
#pragma unroll
        for (int k = 0; k < N; ++k) gprev[k] = g[k], qD[k] = qU[k], fyD[k] = fyU[k];
        lyD = lyU;
    }
}

// FUSE, phase 1 -- row r along x: BOTH axes of its interior cells once (the
// y-flux / y wave speed published for their column's warp), the x-axis of
// its two x-halo cells, the x-faces and x-updates (acc); plus the y-axis of
// column r's two y-halo cells (kept for phase 2).
template <class R, int P, class Eq, int N>
__device__ __forceinline__ void row_fused(const Eq& eq, const Cells<P, N>& c, int r, double s, double (&acc)[P][N],
                                          double (&fyh)[2][N], double (&lyh)[2], bool& bad) {
    double qL[N], fxL[N], lxL, gprev[N], d[N], dl;
    c.load(-1, r, qL);
    pencil::eval<R, true, false>(eq, qL, fxL, lxL, d, dl, bad);
#pragma unroll
    for (int x = 0; x <= P; ++x) {
        double qR[N], fxR[N], lxR, g[N];
        c.load(x, r, qR);
        if (x < P) {
            double fy[N], ly;
            pencil::eval<R, true, true>(eq, qR, fxR, lxR, fy, ly, bad);
#pragma unroll
            for (int k = 0; k < N; ++k) c.at(k, x, r) = fy[k];
            c.at(N, x, r) = ly;
        } else {
            pencil::eval<R, true, false>(eq, qR, fxR, lxR, d, dl, bad);
        }
        pencil::face<R>(qL, qR, fxL, fxR, lxL, lxR, g);  // x-face at x - 1/2
        if (x > 0) {
#pragma unroll
            for (int k = 0; k < N; ++k) acc[x - 1][k] = qL[k];
            rusanov_update(acc[x - 1], gprev, g, s);
        }
#pragma unroll
        for (int k = 0; k < N; ++k) gprev[k] = g[k], qL[k] = qR[k], fxL[k] = fxR[k];
        lxL = lxR;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // column r's y-halo cells (r, -1), (r, P)
        double q[N];
        c.load(r, h == 0 ? -1 : P, q);
        pencil::eval<R, false, true>(eq, q, d, dl, fyh[h], lyh[h], bad);
    }
}

// FUSE, phase 2 -- column r along y: its p+1 y-faces from the published
// fluxes, the differences G_{y-1/2} - G_{y+1/2} written over the fluxes of
// the same cells (each cell's flux is read before its slot is rewritten).
template <class R, int P, int N>
__device__ __forceinline__ void col_faces(const Cells<P, N>& c, int r, const double (&fyh)[2][N],
                                          const double (&lyh)[2]) {
    double qD[N], fyD[N], lyD = lyh[0], gprev[N];
    c.load(r, -1, qD);
#pragma unroll
    for (int k = 0; k < N; ++k) fyD[k] = fyh[0][k];
#pragma unroll
    for (int y = 0; y <= P; ++y) {
        double qU[N], fyU[N], lyU, g[N];
        c.load(r, y, qU);
        if (y < P) {
#pragma unroll
            for (int k = 0; k < N; ++k) fyU[k] = c.at(k, r, y);
            lyU = c.at(N, r, y);
        } else {
#pragma unroll
            for (int k = 0; k < N; ++k) fyU[k] = fyh[1][k];
            lyU = lyh[1];
        }
        pencil::face<R>(qD, qU, fyD, fyU, lyD, lyU, g);  // y-face at y - 1/2
        if (y > 0) {
#pragma unroll
            for (int k = 0; k < N; ++k) c.at(k, r, y - 1) = gprev[k] - g[k];
        }
#pragma unroll
        for (int k = 0; k < N; ++k) gprev[k] = g[k], qD[k] = qU[k], fyD[k] = fyU[k];
        lyD = lyU;
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

template <int P, int N, int NB, bool FUSE>
constexpr size_t tile_smem() {
    return sizeof(tile::CtaSmem<P, N, NB, FUSE>);
}

// CTA = P warps; group g (32 patches from t0 + 32 g) for g = blockIdx.x,
// + gridDim.x, ...  Warp r owns row r and column r of every patch of the
// group.  The host guarantees 16-byte aligned segments.
template <class Eq, int P, int RED, int MINB, int NB, bool FUSE>
__global__ void __launch_bounds__(32 * P, MINB) fused2d_tile_kernel(StepArgs a) {
    using namespace tile;
    constexpr int N = Eq::kUnknowns;
    constexpr int TH = 32 * P;
    using Gm = Geo<P, N>;
    static_assert(Eq::kDim == 2, "2D patches");
    static_assert(RED != kReduceFiltered || kHasLambdaBelow<Eq>, "filtered reduction needs lambda_below");
    const Eq eq(a.gamma);

    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto& S = *reinterpret_cast<CtaSmem<P, N, NB, FUSE>*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31;
    const int r = tid >> 5;  // this warp's row and column (warp-uniform)
    const long long t0 = a.t0, t1 = a.t1;
    const long long groups = (t1 - t0 + G - 1) / G;
    const double scale = step_scale(a);
    const bool fast = step_fast(a, scale);

    auto issue_load = [&](long long g, int b) {  // thread 0: the group's N input segments into buffer b
        const long long first = t0 + g * G;
        const unsigned bytes = (unsigned)(min((long long)G, t1 - first) * Gm::M * 8);
        slab::mbar_expect_tx(&S.mbar[b], N * bytes);
#pragma unroll
        for (int k = 0; k < N; ++k)
            slab::bulk_g2s(&S.in[b][k][0], a.q_in + k * a.in.k + first * Gm::M, bytes, &S.mbar[b]);
    };

    if (tid == 0) {
#pragma unroll
        for (int b = 0; b < NB; ++b) slab::mbar_init(&S.mbar[b], 1);
        slab::fence_mbar_init();
    }
    __syncthreads();
    long long g = blockIdx.x;
    if (tid == 0 && g < groups) issue_load(g, 0);
    int buf = 0;

    double red = 0.0;
    LamFilter lf;
    lf.init();
    unsigned phase = 0;  // bit b: parity of buffer b's next completion
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
        const Cells<P, N> c{&S.in[buf][0][(valid ? lane : 0) * Gm::M], &S.out[0][lane * Gm::Mi]};
        if (tid == 0) bulk_wait_read();  // the previous group's stores have read `out`
        __syncthreads();
        if (NB == 2 && tid == 0 && g + gridDim.x < groups) issue_load(g + gridDim.x, buf ^ 1);  // the other buffer is free
        slab::mbar_wait(&S.mbar[buf], (phase >> buf) & 1u);
        phase ^= 1u << buf;

        // ---- row r along x, column r along y (fast path; IEEE redo if any
        // state of the group is uncertified)
        double acc[P][N];
        bool fold = false;
        if constexpr (FUSE) {  // every cell's microkernels once; the column faces after a barrier
            double fyh[2][N], lyh[2];
            if constexpr (kHasFastPath<Eq>) {
                bool bad = !lane_fast;
                row_fused<XReal>(eq, c, r, 0.5 * s, acc, fyh, lyh, bad);
                fold = !slab::slot_any(1, TH, bad && valid);  // also the barrier after phase 1
            } else {
                __syncthreads();
            }
            if (!fold) {
                bool unused = false;
                row_fused<double>(eq, c, r, s, acc, fyh, lyh, unused);
                __syncthreads();
            }
            if (fold) col_faces<XReal>(c, r, fyh, lyh);
            else col_faces<double>(c, r, fyh, lyh);
            __syncthreads();
        } else {
            if constexpr (kHasFastPath<Eq>) {
                bool bad = !lane_fast;
                y_col<XReal>(eq, c, r, bad);  // first: its results go to shared memory,
                x_row<XReal>(eq, c, r, 0.5 * s, acc, bad);  // acc stays live only across the barrier
                fold = !slab::slot_any(1, TH, bad && valid);  // also the barrier after the passes
            } else {
                __syncthreads();
            }
            if (!fold) {
                bool unused = false;
                y_col<double>(eq, c, r, unused);
                x_row<double>(eq, c, r, s, acc, unused);
                __syncthreads();
            }
        }
        if (NB == 1 && tid == 0 && g + gridDim.x < groups) issue_load(g + gridDim.x, 0);  // `in` is free
        if (NB == 2) buf ^= 1;
        // ---- row r finished: acc_x + s * (G_l - G_r), the reference's order
        const double sf = fold ? 0.5 * s : s;
#pragma unroll
        for (int x = 0; x < P; ++x)
#pragma unroll
            for (int k = 0; k < N; ++k) {
                acc[x][k] = acc[x][k] + sf * c.at(k, x, r);
                c.at(k, x, r) = acc[x][k];
            }
        // every writer orders its generic writes of `out` before the async
        // proxy's bulk stores (CUTLASS's TMA-store convention), then the CTA
        // barrier hands them to the storing thread.  (Letting the other warps
        // skip the wait with bar.arrive measured 1% slower.)
        fence_async_shared();
        __syncthreads();
        if (tid == 0) {
            const unsigned bytes = (unsigned)(np * Gm::Mi * 8);
#pragma unroll
            for (int k = 0; k < N; ++k) bulk_s2g(a.q_out + k * a.out.k + first * Gm::Mi, &S.out[k][0], bytes);
            bulk_commit();
        }

        // ---- reduce over row r's finished cells
        double pred = 0.0;
        if constexpr (RED == kReduceAll) {
#pragma unroll
            for (int x = 0; x < P; ++x) running_max(pred, lambda_of(eq, acc[x]));
        } else if constexpr (RED == kReduceFiltered) {  // only cells the policy cannot place under tau
            bool need[P], any = false;
#pragma unroll
            for (int x = 0; x < P; ++x) any |= need[x] = valid && !eq.lambda_below(acc[x], lf.tau_lo);
            if (__any_sync(0xffffffffu, any)) {
#pragma unroll
                for (int x = 0; x < P; ++x)
                    if (need[x]) running_max(pred, lambda_of(eq, acc[x]));
                lf.raise(pred);
            }
        }
        if constexpr (RED != kReduceNone) {
            if (!valid) pred = 0.0;
            running_max(red, pred);
            if (RED == kReduceAll && a.lam_patch != nullptr) {  // the patch's max over the P rows
                S.red[r][lane] = pred;
                __syncthreads();
                if (r == 0 && valid) {
                    double v = pred;
#pragma unroll
                    for (int w = 1; w < P; ++w) running_max(v, S.red[w][lane]);
                    a.lam_patch[patch] = v;
                }
            }
        }
    }
    if (tid == 0) bulk_wait_all();
    if (RED != kReduceNone && a.lam_bits != nullptr) reduce_epilogue<true>(a, red);
}

}  // namespace fvb
