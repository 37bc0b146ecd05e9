// cascade.cuh -- the "sequence of for-loops" flavour: one data-parallel
// kernel per algorithmic step, stream-ordered, mirroring run_batched
// (pkg/src/patchbench/executors.py:312-382): copy, flux_0..d-1,
// lambda_0..d-1, acc_0..d-1, reduce, each a flat T x range index space with
// a global wait (kernel boundary) after it.  The batch arrays may be in any
// layout (StepArgs::in / out strides); the scratch temporaries are SoA.
//
// Scratch is tight: the axis-a flux temporary holds N*T*(p+2)*p^(d-1)
// doubles and the wave-speed temporary T*(p+2)*p^(d-1) (the reference sizes
// both for the full haloed cube, microkernels.py:70-77 / SPEC.md:149; the
// entries outside the flux range are never read there either).  Scratch
// index of a cell in axis a's range: canonical order of that range,
// coordinate 0 fastest, c_a in [-1,p] and the others in [0,p).
// Every kernel is templated on the physics policy (physics.cuh).
#pragma once

#include "common.cuh"
#include "physics.cuh"

namespace fvb {

// Decode a flat interior index li (coordinate 0 fastest) into coordinates.
template <int D>
__device__ __forceinline__ void interior_coords(int li, int p, int (&c)[D]) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
        c[k] = li % p;
        li /= p;
    }
}

template <int D>
__device__ __forceinline__ int haloed_lin(const int (&c)[D], int m) {
    int lin = 0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) lin = lin * m + (c[k] + 1);
    return lin;
}

// Index of (interior coords c shifted by `shift` along `axis`) in axis' range.
template <int D>
__device__ __forceinline__ int range_index(const int (&c)[D], int axis, int shift, int p) {
    int r = 0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
        const int ext = (k == axis) ? p + 2 : p;
        const int cc = (k == axis) ? c[k] + shift + 1 : c[k];
        r = r * ext + cc;
    }
    return r;
}

// COPY: Q_new(interior) = Q  (microkernels.py:265-270)
template <class Eq>
__global__ void cascade_copy_kernel(StepArgs a) {
    constexpr int D = Eq::kDim, N = Eq::kUnknowns;
    const int p = a.p, m = p + 2;
    const int M = (int)ipow_d(m, D), Mi = (int)ipow_d(p, D);
    const long long end = a.t1 * Mi;
    (void)M;
    for (long long i = a.t0 * Mi + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < end;
         i += (long long)gridDim.x * blockDim.x) {
        const long long patch = i / Mi;
        const int li = (int)(i - patch * Mi);
        int c[D];
        interior_coords<D>(li, p, c);
        const int lh = haloed_lin<D>(c, m);
#pragma unroll
        for (int k = 0; k < N; ++k) out_base(a, patch)[a.out.in_patch(k, li)] = __ldg(in_base(a, patch) + a.in.in_patch(k, lh));
    }
}

// FLUX_axis (microkernels.py:273-296) or EIGENVALUE_axis (:299-315) over the range.
template <class Eq, bool LAMBDA>
__global__ void cascade_flux_kernel(CascadeArgs ca, int axis) {
    constexpr int D = Eq::kDim, N = Eq::kUnknowns;
    const StepArgs& a = ca.s;
    const Eq eq(a.gamma);
    const int p = a.p, m = p + 2;
    const int R = (p + 2) * (int)ipow_d(p, D - 1);
    const long long total = a.T * R, end = a.t1 * R;
    double* __restrict__ tf = ca.tmp_flux[axis];
    double* __restrict__ tl = ca.tmp_lam[axis];
    for (long long i = a.t0 * R + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < end;
         i += (long long)gridDim.x * blockDim.x) {
        const long long patch = i / R;
        int rest = (int)(i - patch * R), lh = 0, mul = 1;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const int ext = (k == axis) ? m : p;
            const int cc = rest % ext;
            rest /= ext;
            lh += ((k == axis) ? cc : cc + 1) * mul;
            mul *= m;
        }
        double q[N];
        const double* qb = in_base(a, patch);
#pragma unroll
        for (int k = 0; k < N; ++k) q[k] = __ldg(qb + a.in.in_patch(k, lh));
        if (LAMBDA) {
            tl[i] = eq.max_eigenvalue(q, axis);
        } else {
            double f[N];
            eq.flux(q, axis, f);
#pragma unroll
            for (int k = 0; k < N; ++k) tf[k * total + i] = f[k];
        }
    }
}

// ACCUMULATE_axis (microkernels.py:318-345)
template <class Eq>
__global__ void cascade_acc_kernel(CascadeArgs ca, int axis) {
    constexpr int D = Eq::kDim, N = Eq::kUnknowns;
    const StepArgs& a = ca.s;
    const int p = a.p, m = p + 2;
    const int Mi = (int)ipow_d(p, D);
    const int R = (p + 2) * (int)ipow_d(p, D - 1);
    const long long rtotal = a.T * R;
    const double* __restrict__ tf = ca.tmp_flux[axis];
    const double* __restrict__ tl = ca.tmp_lam[axis];
    int stride = 1;
    for (int k = 0; k < axis; ++k) stride *= m;
    for (long long i = a.t0 * Mi + blockIdx.x * (long long)blockDim.x + threadIdx.x;
         i < a.t1 * Mi; i += (long long)gridDim.x * blockDim.x) {
        const long long patch = i / Mi;
        const int li = (int)(i - patch * Mi);
        int c[D];
        interior_coords<D>(li, p, c);
        const long long lv = a.in.in_patch(0, haloed_lin<D>(c, m));
        const long long rv = patch * R + range_index<D>(c, axis, 0, p);
        const long long rl = patch * R + range_index<D>(c, axis, -1, p);
        const long long rr = patch * R + range_index<D>(c, axis, +1, p);
        double qv[N], ql[N], qr[N], fv[N], fl[N], fr[N], gl[N], gr[N], acc[N];
        const long long ls = (long long)stride * a.in.l;
        const long long ov = a.out.in_patch(0, li);
        const double* qb = in_base(a, patch);
        double* ob = out_base(a, patch);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const double* qk = qb + k * a.in.k;
            qv[k] = __ldg(qk + lv);
            ql[k] = __ldg(qk + lv - ls);
            qr[k] = __ldg(qk + lv + ls);
            fv[k] = tf[k * rtotal + rv];
            fl[k] = tf[k * rtotal + rl];
            fr[k] = tf[k * rtotal + rr];
            acc[k] = ob[ov + k * a.out.k];
        }
        const double lamv = tl[rv];
        rusanov_face(ql, qv, fl, fv, tl[rl], lamv, gl);
        rusanov_face(qv, qr, fv, fr, lamv, tl[rr], gr);
        rusanov_update(acc, gl, gr, patch_scale(a, step_scale(a), patch));
#pragma unroll
        for (int k = 0; k < N; ++k) ob[ov + k * a.out.k] = acc[k];
    }
}

// REDUCE (microkernels.py:348-361 + executors.py:162-183): grid-wide max of
// max_n lambda_n(Q_new); per-patch maxima via 64-bit atomicMax on the
// zero-initialised lam_patch bits.
template <class Eq, int THREADS>
__global__ void __launch_bounds__(THREADS) cascade_reduce_kernel(StepArgs a) {
    constexpr int D = Eq::kDim, N = Eq::kUnknowns;
    __shared__ double sRed[THREADS / 32];
    const Eq eq(a.gamma);
    const int p = a.p;
    const int Mi = (int)ipow_d(p, D);
    double red = 0.0;
    for (long long i = a.t0 * Mi + blockIdx.x * (long long)THREADS + threadIdx.x; i < a.t1 * Mi;
         i += (long long)gridDim.x * THREADS) {
        const long long patch = i / Mi;
        const double* ob = out_base(a, patch) + a.out.in_patch(0, i - patch * Mi);
        double q[N];
#pragma unroll
        for (int k = 0; k < N; ++k) q[k] = ob[k * a.out.k];
        const double v = cell_max_eigenvalue(eq, q);
        running_max(red, v);
        if (a.lam_patch != nullptr)
            atomic_max_nonneg(reinterpret_cast<unsigned long long*>(a.lam_patch) + i / Mi, v);
    }
    red = block_max<THREADS>(red, sRed);
    if (threadIdx.x == 0 && a.lam_bits != nullptr) atomic_max_nonneg(a.lam_bits, red);
}

}  // namespace fvb
