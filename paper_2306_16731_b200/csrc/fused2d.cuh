// fused2d.cuh -- the nested-parallel ("patch-wise") flavour for 2D patches:
// one warp owns G = 32/P patches at a time, one lane per interior column.
//
// Reference realisation: run_patchwise (pkg/src/patchbench/executors.py:390-445)
// runs every step of a patch inside one parallel region over the union range
// [-1,p]^d with masks.  Here the whole step chain of a patch (copy, flux_x,
// flux_y, lambda_x, lambda_y, acc_x, acc_y, reduce) is fused into one pass of
// a column "pencil" walk along y; no scratch ever touches HBM:
//
//   * y-direction: lane x walks rows Y = -1..P, keeping the previous row's
//     state, y-flux, y-wave-speed, x-updated value and lower y-face in
//     registers (two alternating Row sets, so nothing is copied), and every
//     y-face is computed exactly once;
//   * x-direction: the x-face between columns x and x+1 uses the neighbour's
//     x-flux / wave speed / state via warp shuffles and is handed to lane x+1
//     by one more shuffle, so every interior x-face is computed once; the two
//     x-boundary faces of each row (halo column -1 | 0 and P-1 | halo P) are
//     computed up front in "phase H" by lane r for row r and parked in shared
//     memory (1.5 KB per warp);
//   * update order is the reference's: Q + s*dX first (axis 0), then + s*dY;
//   * reduce: max_n lambda_n(Q_new) of every finished cell, shuffle max,
//     one 64-bit atomicMax per warp per launch.
//
// Arithmetic: the group is first computed with R = XReal (CUDA's fp64
// division / sqrt fast paths written out, reciprocal of rho shared, no
// branches); if any lane of the warp saw an operand outside the fast paths'
// range, the whole group is recomputed with R = double (plain IEEE) and the
// stores are overwritten.  Either way every value is the reference's
// expression on the reference's operands, so output and eigenvalue are
// bit-identical to run_sequential (tests/test_gpu_parity.py).
#pragma once

#include "common.cuh"
#include "euler.cuh"

namespace fvb {

namespace pencil {

constexpr int N = 4;

struct Row {
    double q[N];    // state
    double fy[N];   // y-flux
    double ly;      // y-wave speed
    double acc[N];  // Q + s*dX (x-updated value)
    double gy[N];   // lower y-face G_{Y-1/2}
};

// Evaluate the microkernels of one state with scalar type R.
template <class R, bool X, bool Y>
__device__ __forceinline__ void eval(const Euler<2>& eq, const double (&q)[N], double (&fx)[N],
                                     double& lx, double (&fy)[N], double& ly, bool& bad) {
    R s[N];
#pragma unroll
    for (int k = 0; k < N; ++k) s[k] = q[k];
    if (X) {
        R f[N];
        eq.flux(s, 0, f);
        const R l = eq.max_eigenvalue(s, 0);
#pragma unroll
        for (int k = 0; k < N; ++k) fx[k] = val(f[k]), bad |= is_bad(f[k]);
        lx = val(l), bad |= is_bad(l);
    }
    if (Y) {
        R f[N];
        eq.flux(s, 1, f);
        const R l = eq.max_eigenvalue(s, 1);
#pragma unroll
        for (int k = 0; k < N; ++k) fy[k] = val(f[k]), bad |= is_bad(f[k]);
        ly = val(l), bad |= is_bad(l);
    }
}

template <class R>
__device__ __forceinline__ double cell_lambda(const Euler<2>& eq, const double (&q)[N], bool& bad) {
    R s[N];
#pragma unroll
    for (int k = 0; k < N; ++k) s[k] = q[k];
    const R a = eq.max_eigenvalue(s, 0);
    const R b = eq.max_eigenvalue(s, 1);
    bad |= is_bad(a) | is_bad(b);
    return py_max(val(a), val(b));
}

// Per-warp context of one patch group.
template <int P>
struct Ctx {
    const double* __restrict__ qi;  // this lane's patch, haloed input
    double* __restrict__ qo;        // this lane's patch, output
    long long sIn, sOut;            // SoA unknown strides
    double scale;
    int x, hbase;                   // column; smem index of this patch's row 0
    bool valid;
    double* sGL;                    // [N][48] boundary faces (this warp)
    double* sGR;
};

template <int P>
__device__ __forceinline__ void load_row(const Ctx<P>& c, int Y, double (&q)[N]) {
    const double* p = c.qi + (Y + 1) * (P + 2) + c.x + 1;
#pragma unroll
    for (int k = 0; k < N; ++k) q[k] = __ldg(p + k * c.sIn);
}

// x-faces of row Y and the axis-0 update of this lane's cell.
template <int P>
__device__ __forceinline__ void x_update(const Ctx<P>& c, int Y, const double (&q)[N],
                                         const double (&fx)[N], double lx, double (&acc)[N]) {
    double qn[N], fxn[N], gr[N], gl[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        qn[k] = __shfl_down_sync(0xffffffffu, q[k], 1);
        fxn[k] = __shfl_down_sync(0xffffffffu, fx[k], 1);
    }
    const double lxn = __shfl_down_sync(0xffffffffu, lx, 1);
    rusanov_face(q, qn, fx, fxn, lx, lxn, gr);  // face at x + 1/2
    const int h = c.hbase + Y;
#pragma unroll
    for (int k = 0; k < N; ++k)
        if (c.x == P - 1) gr[k] = c.sGR[k * 48 + h];
#pragma unroll
    for (int k = 0; k < N; ++k) gl[k] = __shfl_up_sync(0xffffffffu, gr[k], 1);
#pragma unroll
    for (int k = 0; k < N; ++k)
        if (c.x == 0) gl[k] = c.sGL[k * 48 + h];
#pragma unroll
    for (int k = 0; k < N; ++k) acc[k] = q[k];
    rusanov_update(acc, gl, gr, c.scale);
}

// Finish row Y-1 (its upper y-face just became known): store + reduce.
template <int P, bool REDUCE, class R>
__device__ __forceinline__ void finish(const Ctx<P>& c, const Euler<2>& eq, int Yprev,
                                       const Row& prev, const double (&gy)[N], double& pred,
                                       bool& bad) {
    double qn[N];
#pragma unroll
    for (int k = 0; k < N; ++k) qn[k] = prev.acc[k];
    rusanov_update(qn, prev.gy, gy, c.scale);
    if (c.valid) {
        double* o = c.qo + Yprev * P + c.x;
#pragma unroll
        for (int k = 0; k < N; ++k) __stcs(o + k * c.sOut, qn[k]);
    }
    if (REDUCE) running_max(pred, cell_lambda<R>(eq, qn, bad));
}

// Interior row Y >= 1: prev = row Y-1, cur <- row Y.
template <int P, bool REDUCE, class R>
__device__ __forceinline__ void row_step(const Ctx<P>& c, const Euler<2>& eq, int Y,
                                         const Row& prev, Row& cur, double& pred, bool& bad) {
    load_row(c, Y, cur.q);
    double fx[N], lx, gy[N];
    eval<R, true, true>(eq, cur.q, fx, lx, cur.fy, cur.ly, bad);
    rusanov_face(prev.q, cur.q, prev.fy, cur.fy, prev.ly, cur.ly, gy);  // face at Y - 1/2
    finish<P, REDUCE, R>(c, eq, Y - 1, prev, gy, pred, bad);
#pragma unroll
    for (int k = 0; k < N; ++k) cur.gy[k] = gy[k];
    x_update(c, Y, cur.q, fx, lx, cur.acc);
}

// One patch group: phase H + the walk.  Returns this lane's max eigenvalue.
template <int P, bool REDUCE, class R, bool PAIR>
__device__ __forceinline__ double group(const Ctx<P>& c, const Euler<2>& eq, bool& bad) {
    // ---- phase H: x-boundary faces of row r = x ---------------------------
    {
        const double* row = c.qi + (c.x + 1) * (P + 2);
        double q0[N], q1[N], q2[N], q3[N], f0[N], f1[N], f2[N], f3[N], l0, l1, l2, l3, g[N], d[N], dl;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            q0[k] = __ldg(row + k * c.sIn);
            q1[k] = __ldg(row + k * c.sIn + 1);
            q2[k] = __ldg(row + k * c.sIn + P);
            q3[k] = __ldg(row + k * c.sIn + P + 1);
        }
        eval<R, true, false>(eq, q0, f0, l0, d, dl, bad);
        eval<R, true, false>(eq, q1, f1, l1, d, dl, bad);
        eval<R, true, false>(eq, q2, f2, l2, d, dl, bad);
        eval<R, true, false>(eq, q3, f3, l3, d, dl, bad);
        rusanov_face(q0, q1, f0, f1, l0, l1, g);
#pragma unroll
        for (int k = 0; k < N; ++k) c.sGL[k * 48 + c.hbase + c.x] = g[k];
        rusanov_face(q2, q3, f2, f3, l2, l3, g);
#pragma unroll
        for (int k = 0; k < N; ++k) c.sGR[k * 48 + c.hbase + c.x] = g[k];
    }
    __syncwarp();

    double pred = 0.0;
    Row S0, S1;
    // row -1 (halo): y-flux only
    {
        load_row(c, -1, S0.q);
        double fx[N], lx;
        eval<R, false, true>(eq, S0.q, fx, lx, S0.fy, S0.ly, bad);
    }
    // row 0: nothing to finish yet
    {
        load_row(c, 0, S1.q);
        double fx[N], lx;
        eval<R, true, true>(eq, S1.q, fx, lx, S1.fy, S1.ly, bad);
        rusanov_face(S0.q, S1.q, S0.fy, S1.fy, S0.ly, S1.ly, S1.gy);
        x_update(c, 0, S1.q, fx, lx, S1.acc);
    }
    int Y = 1;
    if (PAIR) {  // two rows per trip through alternating Row sets: no copies
#pragma unroll 1
        for (; Y + 1 < P; Y += 2) {
            row_step<P, REDUCE, R>(c, eq, Y, S1, S0, pred, bad);
            row_step<P, REDUCE, R>(c, eq, Y + 1, S0, S1, pred, bad);
        }
    } else {  // one row per trip: fewer live registers, a Row copy per row
#pragma unroll 1
        for (; Y + 1 < P; Y += 2) {
            row_step<P, REDUCE, R>(c, eq, Y, S1, S0, pred, bad);
            S1 = S0;
            row_step<P, REDUCE, R>(c, eq, Y + 1, S1, S0, pred, bad);
            S1 = S0;
        }
    }
    if (Y < P) row_step<P, REDUCE, R>(c, eq, Y, S1, S0, pred, bad);
    const Row& last = (Y < P) ? S0 : S1;
    // row P (halo): y-flux, top face, finish row P-1
    {
        double q[N], fx[N], lx, fy[N], ly, gy[N];
        load_row(c, P, q);
        eval<R, false, true>(eq, q, fx, lx, fy, ly, bad);
        rusanov_face(last.q, q, last.fy, fy, last.ly, ly, gy);
        finish<P, REDUCE, R>(c, eq, P - 1, last, gy, pred, bad);
    }
    __syncwarp();  // smem faces reused by the next group
    return pred;
}

}  // namespace pencil

template <int P, int WARPS, bool REDUCE, int MINB, bool PAIR = true>
__global__ void __launch_bounds__(WARPS * 32, MINB) fused2d_pencil_kernel(StepArgs a) {
    using namespace pencil;
    constexpr int M = (P + 2) * (P + 2);
    constexpr int Mi = P * P;
    constexpr int G = 32 / P;  // patches per warp
    static_assert(P >= 2 && P <= 32, "pencil kernel covers 2 <= p <= 32");
    static_assert(G * (P + 1) <= 48, "boundary-face smem row too short");
    const Euler<2> eq{a.gamma};

    __shared__ double sG[WARPS][2][N * 48];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int sub = lane / P;
    const bool lane_used = sub < G;
    const long long t0 = a.t0, t1 = a.t1;
    const long long groups = (t1 - t0 + G - 1) / G;

    Ctx<P> c;
    c.sIn = a.T * M;
    c.sOut = a.T * Mi;
    c.scale = a.scale;
    c.x = lane - sub * P;
    // padded rows (no bank conflict between patches); unused lanes (sub == G)
    // get their own slots: max index G*(P+1) + (32 - G*P) - 1 = G + 31 < 48
    c.hbase = sub * (P + 1);
    c.sGL = sG[warp][0];
    c.sGR = sG[warp][1];

    double red = 0.0;
    for (long long g = (long long)blockIdx.x * WARPS + warp; g < groups;
         g += (long long)gridDim.x * WARPS) {
        long long patch = t0 + g * G + (lane_used ? sub : 0);
        c.valid = lane_used && patch < t1;
        if (!c.valid) patch = t0 + g * G;  // compute on a real patch, never store
        c.qi = a.q_in + patch * M;
        c.qo = a.q_out + patch * Mi;

        bool bad = false;
        double pred = group<P, REDUCE, XReal, PAIR>(c, eq, bad);
        if (__any_sync(0xffffffffu, bad)) {  // operand outside the fast paths: IEEE redo
            bool unused = false;
            pred = group<P, REDUCE, double, PAIR>(c, eq, unused);
        }

        if (!c.valid) pred = 0.0;
        running_max(red, pred);
        if (REDUCE && a.lam_patch != nullptr) {  // segmented max over the P lanes of a patch
            double v = pred;
#pragma unroll
            for (int off = 1; off < P; off <<= 1) {
                const double o = __shfl_down_sync(0xffffffffu, v, off);
                if (c.x + off < P) running_max(v, o);
            }
            if (c.valid && c.x == 0) a.lam_patch[patch] = v;
        }
    }
    if (REDUCE && a.lam_bits != nullptr) {
        red = warp_max(red);
        if (lane == 0) atomic_max_nonneg(a.lam_bits, red);
    }
}

}  // namespace fvb
