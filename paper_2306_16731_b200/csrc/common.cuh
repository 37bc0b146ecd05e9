// common.cuh -- shared pieces of the step kernels: launch arguments, the
// Rusanov face / cell update (the reference's accumulate microkernel,
// pkg/src/patchbench/microkernels.py:157-184 and :318-345) and the
// max-eigenvalue reduction helpers (executors.py:140-211, neutral 0.0).
#pragma once

#include <cstdint>

namespace fvb {

// Batch layouts (patchdata.py:49-58, 142-168; codes as _LAYOUT_CODES :57):
//   AoS   value(k, patch, lin) = base[(patch*M + lin)*N + k]
//   SoA   value(k, patch, lin) = base[k*T*M + patch*M + lin]     (the device default)
//   AoSoA value(k, patch, lin) = base[patch*N*M + k*M + lin]
// M = (p+2)^d for the haloed input, p^d for the interior output.  A layout
// is three strides: offset = k*sk + patch*sp + lin*sl.
enum { kLayoutAoS = 0, kLayoutSoA = 1, kLayoutAoSoA = 2 };

struct Lay {
    long long k, p;  // unknown and patch strides
    int l;           // cell stride (1, or N for AoS)
    __host__ __device__ __forceinline__ long long at(int kk, long long patch, long long lin) const {
        return kk * k + patch * p + lin * l;
    }
    // offset inside one patch (relative to its base, see in_base / out_base)
    __host__ __device__ __forceinline__ long long in_patch(int kk, long long lin) const {
        return kk * k + lin * l;
    }
};

__host__ __device__ inline Lay layout_strides(int layout, long long T, long long M, int N) {
    if (layout == kLayoutAoS) return Lay{1, N * M, N};
    if (layout == kLayoutAoSoA) return Lay{M, N * M, 1};
    return Lay{T * M, M, 1};
}

// A self-resetting device slot for a fused launch's eigenvalue maximum
// (reduce_epilogue): no host-side zeroing between launches.
struct RedSlot {
    unsigned long long bits;  // max of the CTAs' maxima (IEEE bits, >= +0.0)
    unsigned int count;       // CTAs done
    unsigned int pad;
};

// Per-launch arguments shared by every flavour.
struct StepArgs {
    const double* __restrict__ q_in;
    double* __restrict__ q_out;
    long long T;                   // patches in the batch arrays (SoA stride = T*M)
    long long t0, t1;              // patch range [t0, t1) this launch processes
    double scale;                  // dt / h, computed once on the host
    double gamma;
    unsigned long long* lam_bits;  // global max eigenvalue as IEEE bits (>= +0.0), or null
    double* lam_patch;             // per-patch max eigenvalue (T doubles), or null
    int p;                         // volumes per axis
    int fast;                      // run parameters allow the fused kernels' fast arithmetic
    int layout;                    // kLayout* of both batch arrays
    Lay in, out;                   // their strides (haloed input, interior output)
    const double* dt_dev;          // device-resident dt (multi-step runs without host sync), or null
    const double* dt_patch;        // local time stepping: dt of every patch of the batch, or null
    double h;                      // mesh width (with dt_dev / dt_patch: scale formed on the device)
    // SHARED transfer mode (memory.py:162-228): T independently allocated
    // per-patch AoS arrays addressed through pointer tables (device arrays
    // of UVA pointers, typically pinned / registered host memory), computed
    // in place -- the ScatteredFieldView of patchdata.py:318-334.  Null for
    // a contiguous batch.  With tables, layout is AoS and the patch stride
    // of `in` / `out` is unused.
    const double* const* in_tab;
    double* const* out_tab;
    int physics;  // FVB_PHYSICS_* policy the host dispatches on (physics.cuh)
    // fused flavour: the launch's reduction slot (reduce_epilogue), or null
    // (then lam_bits was zeroed by the host and the CTAs atomicMax into it);
    // lam_accumulate: fold the result into *lam_bits (atomicMax) instead of
    // storing it (patch-range launches that accumulate over chunks)
    RedSlot* red_slot;
    int lam_accumulate;
};

// Base of one patch's haloed input / interior output: the batch array at
// patch * patch-stride, or the patch's own array from the pointer table.
__device__ __forceinline__ const double* in_base(const StepArgs& a, long long patch) {
    return a.in_tab != nullptr ? a.in_tab[patch] : a.q_in + patch * a.in.p;
}
__device__ __forceinline__ double* out_base(const StepArgs& a, long long patch) {
    return a.out_tab != nullptr ? a.out_tab[patch] : a.q_out + patch * a.out.p;
}

// dt/h of the launch: the host's value, or the same IEEE quotient formed on
// the device from a device-resident dt (fvb_step_dt).
__device__ __forceinline__ double step_scale(const StepArgs& a) {
    return a.dt_dev != nullptr ? __ddiv_rn(*a.dt_dev, a.h) : a.scale;
}
// run parameters allow the fused kernels' fast arithmetic (fvb.cu plan_run)
__device__ __forceinline__ bool step_fast(const StepArgs& a, double scale) {
    if (a.dt_dev == nullptr && a.dt_patch == nullptr) return a.fast != 0;
    return scale >= 0x1p-1000 && scale <= 0x1p+1000 && a.gamma <= 0x1p+100;
}
// Local time stepping (fvb_step_lts): the dt/h of one patch of the batch.
__device__ __forceinline__ double patch_scale(const StepArgs& a, double uniform, long long patch) {
    return a.dt_patch != nullptr ? __ddiv_rn(a.dt_patch[patch], a.h) : uniform;
}

// Cascade / graph flavours: the step arguments plus the per-axis scratch
// temporaries ([k][patch][r] flux, [patch][r] wave speed; see cascade.cuh).
struct CascadeArgs {
    StepArgs s;
    double* tmp_flux[3];
    double* tmp_lam[3];
};

// Python builtin max(a, b) (microkernels.py:177-178): a unless b > a.
__device__ __forceinline__ double py_max(double a, double b) { return (b > a) ? b : a; }

// Face flux between left state L and right state R along one axis,
// F = 0.5*(F_L + F_R) - (0.5*w)*(Q_R - Q_L),  w = max(lam_L, lam_R).
// Both accumulate calls of the reference (left face of R, right face of L)
// evaluate exactly these operands in this order, so computing it once per
// face and sharing it is bit-identical.
template <int N>
__device__ __forceinline__ void rusanov_face(const double (&qL)[N], const double (&qR)[N],
                                             const double (&fL)[N], const double (&fR)[N],
                                             double lamL, double lamR, double (&g)[N]) {
    const double hw = 0.5 * py_max(lamL, lamR);
#pragma unroll
    for (int k = 0; k < N; ++k) g[k] = 0.5 * (fL[k] + fR[k]) - hw * (qR[k] - qL[k]);
}

// Q_new += (dt/h) * (F_left_face - F_right_face)  (microkernels.py:183-184)
template <int N>
__device__ __forceinline__ void rusanov_update(double (&acc)[N], const double (&gl)[N],
                                               const double (&gr)[N], double scale) {
#pragma unroll
    for (int k = 0; k < N; ++k) acc[k] = acc[k] + scale * (gl[k] - gr[k]);
}

// max_n lambda_n(q) with the reference's association (microkernels.py:187-193).
template <class Eq, int N>
__device__ __forceinline__ double cell_max_eigenvalue(const Eq& eq, const double (&q)[N]) {
    double v = eq.max_eigenvalue(q, 0);
#pragma unroll
    for (int a = 1; a < Eq::kDim; ++a) v = py_max(v, eq.max_eigenvalue(q, a));
    return v;
}

// Running max with the sequential executor's comparison (executors.py:263-269):
// only a strictly greater candidate replaces the current value.
__device__ __forceinline__ void running_max(double& red, double v) {
    if (v > red) red = v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, v, off);
        running_max(v, o);
    }
    return v;
}

// Reduction modes of the fused kernels: none, every finished cell's
// eigenvalue evaluated (needed for per-patch maxima), or filtered (only the
// cells the policy's lambda_below hook cannot place under the warp's running maximum).
constexpr int kReduceNone = 0, kReduceAll = 1, kReduceFiltered = 2;

// Per-warp state of the filtered reduction: tau = the largest eigenvalue the
// warp has evaluated exactly (warp-uniform), tau_lo = tau * (1 - 2^-40).
// Skipping a cell whose eigenvalue is certainly below tau cannot change the
// batch maximum, because tau is the eigenvalue of a cell of the batch.
struct LamFilter {
    double tau, tau_lo;
    __device__ __forceinline__ void init() { tau = tau_lo = 0.0; }
    // every lane of the warp calls it with its running maximum
    __device__ __forceinline__ void raise(double v) { raise_max(warp_max(v)); }
    // the vote group's maximum, already reduced (sub-warp slots)
    __device__ __forceinline__ void raise_max(double v) {
        if (v > tau) {
            tau = v;
            tau_lo = v * (1.0 - 0x1p-40);
        }
    }
};

// Global max of non-negative doubles: their IEEE bit patterns order like the
// values, so an unsigned 64-bit atomicMax is an exact max.
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* bits, double v) {
    if (v > 0.0) atomicMax(bits, (unsigned long long)__double_as_longlong(v));
}

// The end of a fused launch: this thread's running maximum `v` into the
// launch's result.  Every thread of the CTA calls it.  With a slot the
// warps' maxima meet in the self-resetting device slot and the CTA that
// finishes last reads it out, resets it and writes the result -- the host
// needs no memset (a launch gap) before the kernel.  Max is exact, so the
// bits equal the atomicMax-on-zeroed-output path.
template <bool CTA_SYNC>
__device__ __forceinline__ void reduce_epilogue(const StepArgs& a, double v) {
    v = warp_max(v);
    const bool lead = (threadIdx.x & 31) == 0;
    if (a.red_slot == nullptr) {
        if (lead) atomic_max_nonneg(a.lam_bits, v);
        return;
    }
    if (lead) {
        atomic_max_nonneg(&a.red_slot->bits, v);
        __threadfence();
    }
    if (CTA_SYNC) __syncthreads();
    else __syncwarp();
    if (threadIdx.x == 0 && atomicAdd(&a.red_slot->count, 1u) == gridDim.x - 1) {
        __threadfence();
        const unsigned long long m = atomicExch(&a.red_slot->bits, 0ull);
        atomicExch(&a.red_slot->count, 0u);
        if (a.lam_accumulate) {
            if (m != 0ull) atomicMax(a.lam_bits, m);
        } else {
            *a.lam_bits = m;
        }
    }
}

// Block-wide max; every thread must call it; result valid in thread 0.
template <int THREADS>
__device__ __forceinline__ double block_max(double v, double* scratch /* THREADS/32 */) {
    v = warp_max(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        double w = (threadIdx.x < THREADS / 32) ? scratch[threadIdx.x] : 0.0;
        v = warp_max(w);
    }
    __syncthreads();
    return v;
}

__device__ __forceinline__ long long ipow_d(long long b, int e) {
    long long r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

}  // namespace fvb
