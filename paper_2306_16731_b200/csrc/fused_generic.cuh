// fused_generic.cuh -- nested-parallel ("patch-wise") flavour for any d, p:
// one CTA per patch (grid-stride), the haloed patch staged into shared
// memory once, the per-axis flux / wave-speed temporaries of the reference
// (ScratchArrays, pkg/src/patchbench/microkernels.py:70-112) kept in shared
// memory one axis at a time, the output accumulated in shared memory and
// stored once.  This is the 3D kernel (d=3, p=8: 108 KB smem, 2 CTAs/SM) and
// the fallback for 2D patches the pencil kernel does not cover (p > 32).
//
// Per patch it runs the reference's step sequence (kernelgraph.py:173-182)
// with a __syncthreads between dependent steps, exactly like
// run_patchwise (executors.py:390-445) runs them per patch with masks; the
// flux and wave-speed of an axis share one pass (same range, same state).
#pragma once

#include "common.cuh"
#include "physics.cuh"

namespace fvb {

// Shared-memory doubles the generic kernel needs for one patch:
// Q (N*M) + F_axis (N*M) + lambda_axis (M) + Q_new (N*Mi)  [+ reduction scratch]
__host__ __device__ inline long long generic_smem_doubles(int d, int p) {
    long long m = p + 2, M = 1, Mi = 1;
    for (int i = 0; i < d; ++i) M *= m, Mi *= p;
    const int n = d + 2;
    return n * M + n * M + M + n * Mi + 32;
}

template <class Eq, int THREADS, bool REDUCE>
__global__ void __launch_bounds__(THREADS) fused_generic_kernel(StepArgs a) {
    constexpr int D = Eq::kDim, N = Eq::kUnknowns;
    extern __shared__ double smem[];
    const Eq eq(a.gamma);
    const int p = a.p, m = p + 2;
    const int M = (int)ipow_d(m, D), Mi = (int)ipow_d(p, D);

    double* sQ = smem;       // [k][lin_h]
    double* sF = sQ + N * M;  // [k][lin_h], current axis
    double* sL = sF + N * M;  // [lin_h], current axis
    double* sO = sL + M;      // [k][lin_i]
    double* sRed = sO + N * Mi;
    const double uniform_scale = step_scale(a);
    double red = 0.0;

    for (long long patch = a.t0 + blockIdx.x; patch < a.t1; patch += gridDim.x) {
        const double scale = patch_scale(a, uniform_scale, patch);
        // stage the haloed patch (N contiguous segments of M doubles)
        for (int i = threadIdx.x; i < N * M; i += THREADS) {
            const int k = i / M, lin = i - k * M;
            sQ[i] = __ldg(in_base(a, patch) + a.in.in_patch(k, lin));
        }
        __syncthreads();
        // COPY (microkernels.py:124-126)
        for (int li = threadIdx.x; li < Mi; li += THREADS) {
            int rest = li, lh = 0, mul = 1;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const int cc = rest % p;
                rest /= p;
                lh += (cc + 1) * mul;
                mul *= m;
            }
#pragma unroll
            for (int k = 0; k < N; ++k) sO[k * Mi + li] = sQ[k * M + lh];
        }
#pragma unroll 1
        for (int axis = 0; axis < D; ++axis) {
            // FLUX_axis + EIGENVALUE_axis over c_axis in [-1,p], others [0,p)
            int range = 1;
            for (int c = 0; c < D; ++c) range *= (c == axis) ? m : p;
            for (int r = threadIdx.x; r < range; r += THREADS) {
                int rest = r, lh = 0, mul = 1;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const int ext = (c == axis) ? m : p;
                    const int cc = rest % ext;
                    rest /= ext;
                    lh += (c == axis ? cc : cc + 1) * mul;
                    mul *= m;
                }
                double q[N], f[N];
#pragma unroll
                for (int k = 0; k < N; ++k) q[k] = sQ[k * M + lh];
                eq.flux(q, axis, f);
#pragma unroll
                for (int k = 0; k < N; ++k) sF[k * M + lh] = f[k];
                sL[lh] = eq.max_eigenvalue(q, axis);
            }
            __syncthreads();
            // ACCUMULATE_axis (microkernels.py:157-184)
            int stride = 1;
            for (int c = 0; c < axis; ++c) stride *= m;
            for (int li = threadIdx.x; li < Mi; li += THREADS) {
                int rest = li, lv = 0, mul = 1;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const int cc = rest % p;
                    rest /= p;
                    lv += (cc + 1) * mul;
                    mul *= m;
                }
                const int ll = lv - stride, lr = lv + stride;
                double qv[N], ql[N], qr[N], fv[N], fl[N], fr[N], gl[N], gr[N], acc[N];
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    qv[k] = sQ[k * M + lv];
                    ql[k] = sQ[k * M + ll];
                    qr[k] = sQ[k * M + lr];
                    fv[k] = sF[k * M + lv];
                    fl[k] = sF[k * M + ll];
                    fr[k] = sF[k * M + lr];
                    acc[k] = sO[k * Mi + li];
                }
                const double lamv = sL[lv];
                rusanov_face(ql, qv, fl, fv, sL[ll], lamv, gl);
                rusanov_face(qv, qr, fv, fr, lamv, sL[lr], gr);
                rusanov_update(acc, gl, gr, scale);
#pragma unroll
                for (int k = 0; k < N; ++k) sO[k * Mi + li] = acc[k];
            }
            __syncthreads();
        }
        // store + REDUCE (microkernels.py:187-193)
        double pred = 0.0;
        for (int i = threadIdx.x; i < N * Mi; i += THREADS) {
            const int k = i / Mi, li = i - k * Mi;
            __stcs(out_base(a, patch) + a.out.in_patch(k, li), sO[i]);
        }
        if (REDUCE) {
            for (int li = threadIdx.x; li < Mi; li += THREADS) {
                double q[N];
#pragma unroll
                for (int k = 0; k < N; ++k) q[k] = sO[k * Mi + li];
                running_max(pred, cell_max_eigenvalue(eq, q));
            }
            pred = block_max<THREADS>(pred, sRed);
            if (threadIdx.x == 0) {
                running_max(red, pred);
                if (a.lam_patch != nullptr) a.lam_patch[patch] = pred;
            }
        } else {
            __syncthreads();
        }
    }
    // every thread reaches this point (the patch loop is CTA-uniform); only
    // thread 0 holds the CTA's maximum, the others contribute 0
    if (REDUCE && a.lam_bits != nullptr) reduce_epilogue<true>(a, threadIdx.x == 0 ? red : 0.0);
}

}  // namespace fvb
