// fused3d_warp.cuh -- 3D plane walk with ONE warp per patch (p = 8).
//
// Same algorithm, smem layout and TMA plane ring as fused3d.cuh, but the 64
// interior columns of a patch belong to one warp: lane l owns the two
// vertically adjacent columns (x, y) and (x, y+1) with x = l % 8 and
// y = {0, 4, 2, 6}[l / 8] (a half-warp then covers rows y and y+4 for
// either cell, which keeps its 64-bit shared-memory accesses conflict-free,
// see cell_of in fused3d.cuh).  Consequences:
//   * no named barriers: the in-plane exchange needs only __syncwarp, so no
//     warp waits for another warp's halo / boundary-face share;
//   * the halo work is exactly one cell per lane (4p = 32 halo cells);
//   * the y-face between a lane's two cells is formed in registers;
//   * two independent cell chains per lane (ILP) instead of one;
//   * each z-plane (all N unknowns) arrives with ONE tensor-map TMA copy
//     (4-D map [lin][plane][k][patch] over the batch, host-encoded per launch,
//     fvb_plane_map in slab3d.cu) issued from a running (patch, plane)
//     counter -- no per-unknown bulk copies, no 64-bit job division.
// Reference realisation: run_patchwise (pkg/src/patchbench/executors.py:390-445);
// arithmetic and the IEEE redo as in fused3d.cuh, bit-identical to
// run_sequential.
#pragma once

#include <cuda.h>  // CUtensorMap

#include "fused3d.cuh"

namespace fvb {

namespace slabw {

using namespace slab;

// Plane (patch, plane) of the batch -> ring slot, all N unknowns in one
// tensor-map copy completing on the slot's mbarrier.  The map's dimensions
// are ordered by stride: [lin][plane][patch][k] (SoA) or [lin][plane][k][patch]
// (AoSoA), box {M2, 1, N, 1}, coordinates {0, plane, c2, c3} with (c2, c3) =
// (patch, 0) or (0, patch); AoS: the plane's N*M2 interleaved doubles as
// [M2][N][plane][patch], box {M2, N, 1, 1}, coordinates {0, 0, plane, patch}
// (the slot then holds the plane in memory order, [lin][k]).
__device__ __forceinline__ void tma_plane(void* dst, const CUtensorMap* tm, int c1, int c2, int c3,
                                          unsigned long long* m) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(tm)), "r"(0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(m))
        : "memory");
}

// Shared memory of one warp: the plane ring, the in-plane fluxes and wave
// speeds as 16-byte-aligned RECORDS per cell ([lin][flux_0..N-1, wave
// speed, pad]: a neighbour's whole record in (N+1)/2 128-bit loads instead
// of N+1 64-bit ones; a quarter-warp of lanes reading consecutive cells of
// a row hits distinct banks at the 48-byte stride), and the faces.
// The exchange arrays hold only the in-plane indices hlin(x, y) they are
// addressed with (the accessors take the haloed index): x-records x in
// [-1, P], y in [0, P); y-records x in [0, P), y in [-1, P]; faces x, y in
// [0, P] (gx: y < P; gy: x < P).  p = 8: 23.7 instead of 25.6 KB per warp.
template <int P, int RING, int N>
struct alignas(128) WarpSmem {
    static constexpr int E = P + 2;
    static constexpr int NP = (N + 2) / 2 * 2;  // record length in doubles (even)
    static constexpr int FX0 = E, FXN = E * P;        // hlin(-1, 0) .. hlin(P, P-1)
    static constexpr int FY0 = 1, FYN = E * E - 2;    // hlin(0, -1) .. hlin(P-1, P)
    static constexpr int G0 = E + 1, GN = E * P + P;  // hlin(0, 0) .. hlin(P-1, P), covers hlin(P, P-1)
    RingSlot<P, N> ring[RING];
    double fxl_[FXN][NP];  // x-flux and x wave speed of each in-plane cell
    double fyl_[FYN][NP];  // y-flux and y wave speed
    double gx_[N][GN];     // left x-face of cell (x, y), x in [0, P]
    double gy_[N][GN];     // lower y-face of cell (x, y), y in [0, P]
    unsigned long long mbar[RING];
    __device__ __forceinline__ double* fxl(int i) { return fxl_[i - FX0]; }
    __device__ __forceinline__ double* fyl(int i) { return fyl_[i - FY0]; }
    __device__ __forceinline__ double& gx(int k, int i) { return gx_[k][i - G0]; }
    __device__ __forceinline__ double& gy(int k, int i) { return gy_[k][i - G0]; }
};

// The next plane job to issue (jobs are issued strictly in order).
struct TmaIssue {
    int patch, plane;  // batch patch index, plane 0..P+1
    long long left;    // jobs still to issue
};

// The warp's plane ring fed by tensor-map copies: job j lives in slot j % RING.
// LS = N: AoS planes (cells N apart in the slot).
template <int P, int RING, int N, int LS = 1>
struct TmaWalk {
    WarpSmem<P, RING, N>* S;
    const CUtensorMap* tm;
    long long& j;
    TmaIssue& is;
    int lane, stride;
    bool patch_d2;  // the map's patch dimension is 2 (else 3)

    // issue the next job into ring slot r (every lane calls it; lane 0 copies)
    __device__ __forceinline__ void issue(int r) const {
        if (lane == 0) {
            mbar_expect_tx(&S->mbar[r], N * Geo3<P>::M2 * 8);
            if constexpr (LS != 1) {
                tma_plane(&S->ring[r].v[0][0], tm, 0, is.plane, is.patch, &S->mbar[r]);
            } else {
                tma_plane(&S->ring[r].v[0][0], tm, is.plane, patch_d2 ? is.patch : 0, patch_d2 ? 0 : is.patch,
                          &S->mbar[r]);
            }
        }
        if (++is.plane == P + 2) {
            is.plane = 0;
            is.patch += stride;
        }
        --is.left;
    }
    __device__ __forceinline__ Plane<LS> acquire() const {
        const int r = (int)(j % RING);
        mbar_wait(&S->mbar[r], (unsigned)((j / RING) & 1));
        return Plane<LS>{&S->ring[r].v[0][0], LS == 1 ? Geo3<P>::M2 : 1};
    }
    // every lane is done reading the current slot (after __syncwarp)
    __device__ __forceinline__ void release() const {
        if (is.left > 0) {  // no proxy fence: reads ordered by the __syncwarp before release()
            issue((int)(j % RING));
        }
        ++j;
    }
};

// Carried along z for the lane's two columns.
template <int N>
struct Carry2 {
    Carry<N> a, b;
};

template <int P, int RING, int LS, int N>
struct WarpCtx {
    SlabCtx<P, RING, LS, N> s;  // stream / strides / duties (s.t = lane; s.S unused)
    WarpSmem<P, RING, N>* W;    // the warp's ring, flux records and faces
    int lcA, ciA;            // haloed / interior in-plane index of cell A; B is one row up
};

// One interior plane z for the warp.  Phase 1: evaluate both cells (publish
// in-plane fluxes), the lane's halo cell, the z-faces below, finish (x, y,
// z-1) and (x, y+1, z-1).  Phase 2: left x-faces of both cells, the lower
// y-face of A (the A|B face stays in registers), boundary faces.  Phase 3:
// right faces, x/y updates.
template <int P, int RING, int RED, class R, class W, int LS, class Eq, int N>
__device__ __forceinline__ void warp_plane(const WarpCtx<P, RING, LS, N>& w, const W& walk, const Eq& eq,
                                           int z, const Carry2<N>& prev, Carry2<N>& cur, double* qo, double& pred,
                                           LamFilter& lf, bool& bad) {
    using Gm = Geo3<P>;
    constexpr int E = Gm::E, CELLS = Gm::CELLS;
    const SlabCtx<P, RING, LS, N>& c = w.s;
    WarpSmem<P, RING, N>& S = *w.W;
    constexpr int NP = WarpSmem<P, RING, N>::NP;
    const double s = kFold<R> ? c.hscale : c.scale;
    const auto pl = walk.acquire();
    const int la = w.lcA, lb = w.lcA + E;

    // ---- phase 1 -----------------------------------------------------------
    double fyA[N], lyA, fyB[N], lyB;  // kept for the in-register A|B y-face
    {
        double fx[N], lx;
#pragma unroll
        for (int k = 0; k < N; ++k) cur.a.q[k] = pl(k, la);
        R sr[N];
        to_r(cur.a.q, sr);
        certify(eq, sr, bad);
        axis_eval(eq, sr, 0, fx, lx);
        axis_eval(eq, sr, 1, fyA, lyA);
        axis_eval(eq, sr, 2, cur.a.fz, cur.a.lz);
        put_rec<NP>(S.fxl(la), fx, lx);
        put_rec<NP>(S.fyl(la), fyA, lyA);
    }
    {
        double fx[N], lx;
#pragma unroll
        for (int k = 0; k < N; ++k) cur.b.q[k] = pl(k, lb);
        R sr[N];
        to_r(cur.b.q, sr);
        certify(eq, sr, bad);
        axis_eval(eq, sr, 0, fx, lx);
        axis_eval(eq, sr, 1, fyB, lyB);
        axis_eval(eq, sr, 2, cur.b.fz, cur.b.lz);
        put_rec<NP>(S.fxl(lb), fx, lx);
        put_rec<NP>(S.fyl(lb), fyB, lyB);
    }
    {  // the lane's halo cell
        double h[N], f[N], l;
#pragma unroll
        for (int k = 0; k < N; ++k) h[k] = pl(k, c.hl);
        R sr[N];
        to_r(h, sr);
        certify(eq, sr, bad);
        if (c.haxis == 0) {
            axis_eval(eq, sr, 0, f, l);
            put_rec<NP>(S.fxl(c.hl), f, l);
        } else {
            axis_eval(eq, sr, 1, f, l);
            put_rec<NP>(S.fyl(c.hl), f, l);
        }
    }
    face<R>(prev.a.q, cur.a.q, prev.a.fz, cur.a.fz, prev.a.lz, cur.a.lz, cur.a.gz);  // z - 1/2
    face<R>(prev.b.q, cur.b.q, prev.b.fz, cur.b.fz, prev.b.lz, cur.b.lz, cur.b.gz);
    if (z >= 1) {  // finish both cells of plane z-1
        double qn[N];
#pragma unroll
        for (int k = 0; k < N; ++k) qn[k] = prev.a.acc[k];
        rusanov_update(qn, prev.a.gz, cur.a.gz, s);
#pragma unroll
        for (int k = 0; k < N; ++k) __stcs(qo + k * c.sOut + (z - 1) * CELLS * LS, qn[k]);
        reduce_cell<RED, R>(eq, qn, true, pred, lf, bad);
#pragma unroll
        for (int k = 0; k < N; ++k) qn[k] = prev.b.acc[k];
        rusanov_update(qn, prev.b.gz, cur.b.gz, s);
#pragma unroll
        for (int k = 0; k < N; ++k) __stcs(qo + k * c.sOut + ((z - 1) * CELLS + P) * LS, qn[k]);
        reduce_cell<RED, R>(eq, qn, true, pred, lf, bad);
    }
    __syncwarp();

    // ---- phase 2 -----------------------------------------------------------
    double gxlA[N], gxlB[N], gylA[N], gAB[N];
    {
        double qn[N], fn[N], fo[N], ln, lo;
#pragma unroll
        for (int k = 0; k < N; ++k) qn[k] = pl(k, la - 1);
        get_rec<NP>(S.fxl(la - 1), fn, ln);
        get_rec<NP>(S.fxl(la), fo, lo);
        face<R>(qn, cur.a.q, fn, fo, ln, lo, gxlA);
#pragma unroll
        for (int k = 0; k < N; ++k) qn[k] = pl(k, lb - 1);
        get_rec<NP>(S.fxl(lb - 1), fn, ln);
        get_rec<NP>(S.fxl(lb), fo, lo);
        face<R>(qn, cur.b.q, fn, fo, ln, lo, gxlB);
#pragma unroll
        for (int k = 0; k < N; ++k) qn[k] = pl(k, la - E);
        get_rec<NP>(S.fyl(la - E), fn, ln);
        face<R>(qn, cur.a.q, fn, fyA, ln, lyA, gylA);
        face<R>(cur.a.q, cur.b.q, fyA, fyB, lyA, lyB, gAB);  // in registers
#pragma unroll
        for (int k = 0; k < N; ++k) S.gx(k, la) = gxlA[k], S.gx(k, lb) = gxlB[k], S.gy(k, la) = gylA[k];
    }
    if (c.bface) {  // lanes 16..31: right / top boundary faces
        double qL[N], qR[N], fL[N], fR[N], g[N], lL, lR;
        const int bl = c.bl, br = c.bl + c.bstep;
        const double* FL = c.bx ? S.fxl(bl) : S.fyl(bl);
        const double* FR = c.bx ? S.fxl(br) : S.fyl(br);
        double* Gb = c.bx ? &S.gx(0, br) : &S.gy(0, br);  // stride GN per unknown
#pragma unroll
        for (int k = 0; k < N; ++k) {
            qL[k] = pl(k, bl);
            qR[k] = pl(k, br);
        }
        get_rec<NP>(FL, fL, lL);
        get_rec<NP>(FR, fR, lR);
        face<R>(qL, qR, fL, fR, lL, lR, g);
#pragma unroll
        for (int k = 0; k < N; ++k) Gb[k * WarpSmem<P, RING, N>::GN] = g[k];
    }
    __syncwarp();  // faces published; this plane's ring slot no longer read
    walk.release();

    // ---- phase 3 -----------------------------------------------------------
    double gr[N];
#pragma unroll
    for (int k = 0; k < N; ++k) cur.a.acc[k] = cur.a.q[k], gr[k] = S.gx(k, la + 1);
    rusanov_update(cur.a.acc, gxlA, gr, s);
    rusanov_update(cur.a.acc, gylA, gAB, s);
#pragma unroll
    for (int k = 0; k < N; ++k) cur.b.acc[k] = cur.b.q[k], gr[k] = S.gx(k, lb + 1);
    rusanov_update(cur.b.acc, gxlB, gr, s);
#pragma unroll
    for (int k = 0; k < N; ++k) gr[k] = S.gy(k, lb + E);
    rusanov_update(cur.b.acc, gAB, gr, s);
}

template <int P, int RING, int RED, class R, int LS, class Eq, int N>
__device__ __forceinline__ double warp_patch(const WarpCtx<P, RING, LS, N>& w, const TmaWalk<P, RING, N, LS>& walk,
                                             const Eq& eq, long long patch, LamFilter& lf, bool& bad) {
    using Gm = Geo3<P>;
    constexpr int E = Gm::E, CELLS = Gm::CELLS;
    const SlabCtx<P, RING, LS, N>& c = w.s;
    const double s = kFold<R> ? c.hscale : c.scale;
    double* qo = c.q_out + patch * c.pOut + w.ciA * LS;
    double pred = 0.0;
    Carry2<N> A, B;
    {  // z = -1: z-flux only
        const auto pl = walk.acquire();
#pragma unroll
        for (int k = 0; k < N; ++k) A.a.q[k] = pl(k, w.lcA), A.b.q[k] = pl(k, w.lcA + E);
        R sr[N];
        to_r(A.a.q, sr);
        certify(eq, sr, bad);
        axis_eval(eq, sr, 2, A.a.fz, A.a.lz);
        to_r(A.b.q, sr);
        certify(eq, sr, bad);
        axis_eval(eq, sr, 2, A.b.fz, A.b.lz);
        __syncwarp();
        walk.release();
    }
#pragma unroll 1
    for (int z = 0; z < P; z += 2) {
        warp_plane<P, RING, RED, R>(w, walk, eq, z, A, B, qo, pred, lf, bad);
        warp_plane<P, RING, RED, R>(w, walk, eq, z + 1, B, A, qo, pred, lf, bad);
    }
    {  // z = P: top z-faces, finish z = P-1
        const auto pl = walk.acquire();
        double q[N], fz[N], lz, gz[N], qn[N];
        R sr[N];
#pragma unroll
        for (int k = 0; k < N; ++k) q[k] = pl(k, w.lcA);
        to_r(q, sr);
        certify(eq, sr, bad);
        axis_eval(eq, sr, 2, fz, lz);
        face<R>(A.a.q, q, A.a.fz, fz, A.a.lz, lz, gz);
#pragma unroll
        for (int k = 0; k < N; ++k) qn[k] = A.a.acc[k];
        rusanov_update(qn, A.a.gz, gz, s);
#pragma unroll
        for (int k = 0; k < N; ++k) __stcs(qo + k * c.sOut + (P - 1) * CELLS * LS, qn[k]);
        reduce_cell<RED, R>(eq, qn, true, pred, lf, bad);
#pragma unroll
        for (int k = 0; k < N; ++k) q[k] = pl(k, w.lcA + E);
        to_r(q, sr);
        certify(eq, sr, bad);
        axis_eval(eq, sr, 2, fz, lz);
        face<R>(A.b.q, q, A.b.fz, fz, A.b.lz, lz, gz);
#pragma unroll
        for (int k = 0; k < N; ++k) qn[k] = A.b.acc[k];
        rusanov_update(qn, A.b.gz, gz, s);
#pragma unroll
        for (int k = 0; k < N; ++k) __stcs(qo + k * c.sOut + ((P - 1) * CELLS + P) * LS, qn[k]);
        reduce_cell<RED, R>(eq, qn, true, pred, lf, bad);
        __syncwarp();
        walk.release();
    }
    return pred;
}

}  // namespace slabw

// One warp (= one patch slot) per CTA.
template <class Eq, int P, int RING, int RED, int MINB, int LS>
__global__ void __launch_bounds__(32, MINB) fused3d_warp_kernel(StepArgs a, const __grid_constant__ CUtensorMap tm,
                                                                  int patch_d2) {
    using namespace slab;
    using namespace slabw;
    using Gm = Geo3<P>;
    static_assert(Gm::CELLS == 64 && Gm::HALO == 32 && Gm::BULK, "one warp per patch is laid out for p = 8");
    static_assert(Eq::kDim == 3, "the plane walk is 3D");
    static_assert(RED != kReduceFiltered || kHasLambdaBelow<Eq>, "filtered reduction needs lambda_below");
    constexpr int E = Gm::E;
    constexpr int N = Eq::kUnknowns;
    const Eq eq(a.gamma);

    extern __shared__ __align__(128) unsigned char smem_raw[];
    WarpCtx<P, RING, LS, N> w;
    SlabCtx<P, RING, LS, N>& c = w.s;
    const int lane = threadIdx.x;
    c.t = lane;
    c.S = nullptr;
    w.W = reinterpret_cast<WarpSmem<P, RING, N>*>(smem_raw);
    c.bar = 0;
    c.q_in = a.q_in;
    c.q_out = a.q_out;
    c.sIn = a.in.k;
    c.sOut = a.out.k;
    c.pIn = a.in.p;
    c.pOut = a.out.p;
    c.bulk = true;  // unused: planes arrive by the tensor map (TmaWalk)
    const double scale = step_scale(a);
    const bool fast = step_fast(a, scale);
    c.scale = scale;
    c.hscale = 0.5 * scale;
    c.first = a.t0 + (long long)blockIdx.x;
    c.stride = (long long)gridDim.x;
    const long long npatch = c.first < a.t1 ? (a.t1 - c.first + c.stride - 1) / c.stride : 0;
    c.njobs = npatch * (P + 2);

    const int cx = lane % P, g = lane / P;
    const int cy = ((g & 1) << 2) | ((g >> 1) << 1);  // rows {0, 4, 2, 6}: cells (cx, cy), (cx, cy+1)
    w.lcA = hlin<P>(cx, cy);
    w.ciA = cx + P * cy;
    c.real = true;
    c.halo = true;
    {
        const int side = lane / P, i = lane % P;
        const int hx = side == 0 ? -1 : side == 1 ? P : i;
        const int hy = side == 2 ? -1 : side == 3 ? P : i;
        c.hl = hlin<P>(hx, hy);
        c.haxis = side < 2 ? 0 : 1;
    }
    const int b = lane - (32 - Gm::BF);
    c.bface = b >= 0;
    c.bx = b < P;
    const int bi = c.bx ? b : b - P;
    c.bl = c.bface ? (c.bx ? hlin<P>(P - 1, bi) : hlin<P>(bi, P - 1)) : 0;
    c.bstep = c.bx ? 1 : E;

    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < RING; ++r) mbar_init(&w.W->mbar[r], 1);
        fence_mbar_init();
    }
    __syncwarp();
    long long j = 0;
    TmaIssue is{(int)c.first, 0, c.njobs};
    const TmaWalk<P, RING, N, LS> walk{w.W, &tm, j, is, lane, (int)c.stride, patch_d2 != 0};
#pragma unroll
    for (int r = 0; r < RING; ++r)
        if (is.left > 0) walk.issue(r);

    double red = 0.0;
    LamFilter lf;
    lf.init();
    for (long long ip = 0; ip < npatch; ++ip) {
        const long long patch = c.first + ip * c.stride;
        bool patch_fast = fast;
        if (a.dt_patch != nullptr) {  // local time stepping: this patch's dt
            c.scale = patch_scale(a, scale, patch);
            c.hscale = 0.5 * c.scale;
            patch_fast = step_fast(a, c.scale);
        }
        bool bad = !patch_fast;
        const LamFilter lf0 = lf;
        double pred;
        bool redo = false;
        if constexpr (kHasFastPath<Eq>) {
            pred = warp_patch<P, RING, RED, XReal>(w, walk, eq, patch, lf, bad);
            redo = __any_sync(0xffffffffu, bad);
        } else {  // a policy without the fast-path hook: IEEE double throughout
            pred = warp_patch<P, RING, RED, double>(w, walk, eq, patch, lf, bad);
        }
        if (redo) {  // IEEE redo of the patch
            pred = 0.0;
            const double* qi = a.q_in + patch * c.pIn;
#pragma unroll 1
            for (int cell = 0; cell < 2; ++cell) {
                double* qo = a.q_out + patch * c.pOut + (w.ciA + cell * P) * LS;
#pragma unroll 1
                for (int z = 0; z < P; ++z) {
                    double qn[N];
                    redo_cell<P, LS>(eq, qi, c.sIn, cx, cy + cell, z, c.scale, qn);
#pragma unroll
                    for (int k = 0; k < N; ++k) qo[k * c.sOut + z * Gm::CELLS * LS] = qn[k];
                    if (RED != kReduceNone) running_max(pred, cell_max_eigenvalue(eq, qn));
                }
            }
            if (RED == kReduceFiltered) {
                lf = lf0;
                lf.raise(pred);
            }
        }
        running_max(red, pred);
        if (RED == kReduceAll && a.lam_patch != nullptr) {
            const double v = warp_max(pred);
            if (lane == 0) a.lam_patch[patch] = v;
        }
    }
    if (RED != kReduceNone && a.lam_bits != nullptr) reduce_epilogue<false>(a, red);
}

}  // namespace fvb
