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
//     registers, so every y-face is computed exactly once (register carry);
//   * x-direction: the x-face between columns x and x+1 uses the neighbour's
//     x-flux / wave speed / state via warp shuffles and is handed to lane x+1
//     by one more shuffle, so every interior x-face is computed once; the two
//     x-boundary faces of each row (halo column -1 | 0 and P-1 | halo P) are
//     computed up front in "phase H" by lane r for row r and parked in 2 KB of
//     shared memory per warp;
//   * update order is the reference's: Q + s*dX first (axis 0), then + s*dY;
//   * reduce: max_n lambda_n(Q_new) of every finished cell, warp shuffle max,
//     one 64-bit atomicMax per warp per launch.
//
// Every face value is the same expression on the same operands as in the
// reference's accumulate microkernel, so output and eigenvalue are
// bit-identical to run_sequential (checked by tests/test_gpu_parity.py).
#pragma once

#include "common.cuh"
#include "euler.cuh"

namespace fvb {

template <int P, int WARPS, bool REDUCE>
__global__ void __launch_bounds__(WARPS * 32)
    fused2d_pencil_kernel(StepArgs a) {
    constexpr int N = 4;
    constexpr int m = P + 2;
    constexpr int M = m * m;
    constexpr int Mi = P * P;
    constexpr int G = 32 / P;  // patches per warp
    static_assert(P >= 2 && P <= 32, "pencil kernel covers 2 <= p <= 32");
    const Euler<2> eq{a.gamma};

    __shared__ double sGL[WARPS][N][32];  // x-face at -1/2 of row r, by lane (sub*P + r)
    __shared__ double sGR[WARPS][N][32];  // x-face at P-1/2 of row r

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int sub = lane / P;
    const int x = lane - sub * P;
    const bool lane_used = sub < G;
    const long long T = a.T;
    const long long sIn = T * M, sOut = T * Mi;
    const long long t0 = a.t0, t1 = a.t1;
    const long long groups = (t1 - t0 + G - 1) / G;
    const double scale = a.scale;

    double red = 0.0;
    for (long long g = (long long)blockIdx.x * WARPS + warp; g < groups;
         g += (long long)gridDim.x * WARPS) {
        long long patch = t0 + g * G + (lane_used ? sub : 0);
        const bool valid = lane_used && patch < t1;
        if (!valid) patch = t0 + g * G;  // compute on a real patch, never store
        const double* __restrict__ qi = a.q_in + patch * M;
        double* __restrict__ qo = a.q_out + patch * Mi;

        // ---- phase H: x-boundary faces of row r = x -----------------------------
        {
            const int rb = (x + 1) * m;
            double q0[N], q1[N], q2[N], q3[N];
#pragma unroll
            for (int k = 0; k < N; ++k) {
                q0[k] = __ldg(qi + k * sIn + rb);
                q1[k] = __ldg(qi + k * sIn + rb + 1);
                q2[k] = __ldg(qi + k * sIn + rb + P);
                q3[k] = __ldg(qi + k * sIn + rb + P + 1);
            }
            double f0[N], f1[N], g[N];
            eq.flux(q0, 0, f0);
            eq.flux(q1, 0, f1);
            rusanov_face(q0, q1, f0, f1, eq.max_eigenvalue(q0, 0), eq.max_eigenvalue(q1, 0), g);
#pragma unroll
            for (int k = 0; k < N; ++k) sGL[warp][k][lane] = g[k];
            eq.flux(q2, 0, f0);
            eq.flux(q3, 0, f1);
            rusanov_face(q2, q3, f0, f1, eq.max_eigenvalue(q2, 0), eq.max_eigenvalue(q3, 0), g);
#pragma unroll
            for (int k = 0; k < N; ++k) sGR[warp][k][lane] = g[k];
        }
        __syncwarp();

        // ---- walk along y ---------------------------------------------------
        double qp[N], fyp[N], lyp;  // previous row: state, y-flux, y-wave speed
        double accp[N], gyp[N];     // previous row: x-updated value, its lower y-face
        {
#pragma unroll
            for (int k = 0; k < N; ++k) qp[k] = __ldg(qi + k * sIn + x + 1);  // row -1
            eq.flux(qp, 1, fyp);
            lyp = eq.max_eigenvalue(qp, 1);
        }
        double pred = 0.0;  // this lane's max eigenvalue over its finished cells
#pragma unroll 1
        for (int Y = 0; Y <= P; ++Y) {
            double q[N], fy[N], ly, gy[N];
#pragma unroll
            for (int k = 0; k < N; ++k) q[k] = __ldg(qi + k * sIn + (Y + 1) * m + x + 1);
            eq.flux(q, 1, fy);
            ly = eq.max_eigenvalue(q, 1);
            rusanov_face(qp, q, fyp, fy, lyp, ly, gy);  // face at Y - 1/2
            if (Y >= 1) {  // finish row Y-1: + s*(G_{y-1/2} - G_{y+1/2})
                rusanov_update(accp, gyp, gy, scale);
                const int oi = (Y - 1) * P + x;
                if (valid) {
#pragma unroll
                    for (int k = 0; k < N; ++k) __stcs(qo + k * sOut + oi, accp[k]);
                }
                if (REDUCE) running_max(pred, cell_max_eigenvalue(eq, accp));
            }
            const int hrow = (sub * P + Y) & 31;  // lane that parked row Y's boundary faces
            if (Y < P) {  // interior row: x-faces, axis-0 update
                double fx[N], lx, gr[N], gl[N];
                eq.flux(q, 0, fx);
                lx = eq.max_eigenvalue(q, 0);
                double qn[N], fxn[N];
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    qn[k] = __shfl_down_sync(0xffffffffu, q[k], 1);
                    fxn[k] = __shfl_down_sync(0xffffffffu, fx[k], 1);
                }
                const double lxn = __shfl_down_sync(0xffffffffu, lx, 1);
                rusanov_face(q, qn, fx, fxn, lx, lxn, gr);  // face at x + 1/2
                if (x == P - 1) {
#pragma unroll
                    for (int k = 0; k < N; ++k) gr[k] = sGR[warp][k][hrow];
                }
#pragma unroll
                for (int k = 0; k < N; ++k) gl[k] = __shfl_up_sync(0xffffffffu, gr[k], 1);
                if (x == 0) {
#pragma unroll
                    for (int k = 0; k < N; ++k) gl[k] = sGL[warp][k][hrow];
                }
#pragma unroll
                for (int k = 0; k < N; ++k) accp[k] = q[k];
                rusanov_update(accp, gl, gr, scale);
            }
#pragma unroll
            for (int k = 0; k < N; ++k) {
                qp[k] = q[k];
                fyp[k] = fy[k];
                gyp[k] = gy[k];
            }
            lyp = ly;
        }
        __syncwarp();  // sGL/sGR reused by the next group

        if (!valid) pred = 0.0;
        running_max(red, pred);
        if (REDUCE && a.lam_patch != nullptr) {  // segmented max over the P lanes of a patch
            double v = pred;
#pragma unroll
            for (int off = 1; off < P; off <<= 1) {
                const double o = __shfl_down_sync(0xffffffffu, v, off);
                if (x + off < P) running_max(v, o);
            }
            if (valid && x == 0) a.lam_patch[patch] = v;
        }
    }
    if (REDUCE && a.lam_bits != nullptr) {
        red = warp_max(red);
        if (lane == 0) atomic_max_nonneg(a.lam_bits, red);
    }
}

}  // namespace fvb
