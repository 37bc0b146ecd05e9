// misc.cu -- the non-step entry points of the C ABI: seeded synthetic field
// (jump-ahead LCG), AoS<->SoA transfer permutations, microkernel probe and
// admissibility check.
#include "euler.cuh"
#include "host.h"

using namespace fvb;

// ---------------------------------------------------------------------------
// seeded field (bench.py:89-133)
// ---------------------------------------------------------------------------
#define FVB_LCG_A 6364136223846793005ULL
#define FVB_LCG_C 1442695040888963407ULL

__device__ __forceinline__ unsigned long long lcg_jump(unsigned long long s, unsigned long long n) {
    unsigned long long acc_a = 1, acc_c = 0, a = FVB_LCG_A, c = FVB_LCG_C;
    while (n) {
        if (n & 1) {
            acc_a *= a;
            acc_c = acc_c * a + c;
        }
        c = (a + 1) * c;
        a *= a;
        n >>= 1;
    }
    return acc_a * s + acc_c;
}

__device__ __forceinline__ double lcg_uniform(unsigned long long& s, double lo, double hi) {
    s = s * FVB_LCG_A + FVB_LCG_C;
    return lo + (hi - lo) * ((double)(s >> 11) * 0x1p-53);
}

template <int D>
__global__ void init_field_kernel(long long T, long long p0, int p, unsigned long long seed,
                                  double gamma, double* __restrict__ q) {
    constexpr int N = D + 2;
    const long long M = ipow_d(p + 2, D);
    const long long total = T * M;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long patch = i / M, lin = i - patch * M;
        unsigned long long s = lcg_jump(seed, (unsigned long long)(((p0 + patch) * M + lin) * N));
        const double rho = lcg_uniform(s, 0.5, 2.0);
        double u[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < D; ++k) u[k] = lcg_uniform(s, -0.5, 0.5);
        const double pr = lcg_uniform(s, 0.5, 2.0);
        double ke = u[0] * u[0] + u[1] * u[1];
        if (D == 3) ke = ke + u[2] * u[2];
        q[i] = rho;
#pragma unroll
        for (int k = 0; k < D; ++k) q[(1 + k) * total + i] = rho * u[k];
        q[(D + 1) * total + i] = pr / (gamma - 1.0) + 0.5 * rho * ke;
    }
}

extern "C" int fvb_init_field(int dim, int p, int64_t T_local, int64_t patch_begin, uint64_t seed,
                              double gamma, double* q_in_dev, void* stream) {
    int rc = validate_shape(dim, p, T_local);
    if (rc) return rc;
    if (patch_begin < 0) return fail(FVB_EINVAL, "patch_begin must be >= 0");
    const long long total = T_local * ipow_h(p + 2, dim);
    const unsigned grid = (unsigned)blocks_for(total, 256, 16);
    if (dim == 2)
        init_field_kernel<2><<<grid, 256, 0, (cudaStream_t)stream>>>(T_local, patch_begin, p, seed, gamma, q_in_dev);
    else
        init_field_kernel<3><<<grid, 256, 0, (cudaStream_t)stream>>>(T_local, patch_begin, p, seed, gamma, q_in_dev);
    return check_launch("init_field_kernel");
}

// ---------------------------------------------------------------------------
// AoS <-> SoA (memory.py:240-265)
// ---------------------------------------------------------------------------
__global__ void aos_soa_kernel(long long T, long long M, int N, const double* __restrict__ src,
                               double* __restrict__ dst, int to_soa) {
    const long long total = T * M * N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        // i enumerates the SoA array: k slowest, then patch, then lin
        const long long k = i / (T * M), rest = i - k * T * M;  // rest = patch*M + lin
        const long long j = rest * N + k;                          // AoS offset
        if (to_soa) dst[i] = __ldg(src + j);
        else dst[j] = __ldg(src + i);
    }
}

int aos_soa(int dim, int p, int64_t T, int haloed, const double* src, double* dst,
                   void* stream, int to_soa) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    const long long m = haloed ? p + 2 : p, M = ipow_h(m, dim);
    const long long total = T * M * (dim + 2);
    aos_soa_kernel<<<(unsigned)blocks_for(total, 256, 16), 256, 0, (cudaStream_t)stream>>>(
        T, M, dim + 2, src, dst, to_soa);
    return check_launch("aos_soa_kernel");
}

// General re-layout: i enumerates the destination array (coalesced writes).
__global__ void relayout_kernel(long long T, long long M, int N, Lay src_l, Lay dst_l, int dst_layout,
                                const double* __restrict__ src, double* __restrict__ dst) {
    const long long total = T * M * N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        long long k, patch, lin;
        if (dst_layout == kLayoutAoS) {
            k = i % N;
            const long long r = i / N;
            patch = r / M, lin = r - patch * M;
        } else if (dst_layout == kLayoutAoSoA) {
            patch = i / (N * M);
            const long long r = i - patch * N * M;
            k = r / M, lin = r - k * M;
        } else {
            k = i / (T * M);
            const long long r = i - k * T * M;
            patch = r / M, lin = r - patch * M;
        }
        dst[i] = __ldg(src + src_l.at((int)k, patch, lin));
    }
}

extern "C" int fvb_relayout(int dim, int p, int64_t T, int haloed, int src_layout, int dst_layout,
                            const double* src_dev, double* dst_dev, void* stream) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    for (int l : {src_layout, dst_layout})
        if (l != kLayoutAoS && l != kLayoutSoA && l != kLayoutAoSoA)
            return fail(FVB_EINVAL, "unknown layout %d", l);
    if (src_dev == nullptr || dst_dev == nullptr) return fail(FVB_EINVAL, "null batch pointer");
    const long long M = ipow_h(haloed ? p + 2 : p, dim);
    const int N = dim + 2;
    const long long total = T * M * N;
    if (src_layout == dst_layout)
        return cudaMemcpyAsync(dst_dev, src_dev, total * 8, cudaMemcpyDeviceToDevice,
                               (cudaStream_t)stream) == cudaSuccess
                   ? FVB_OK
                   : fail(FVB_ECUDA, "relayout copy failed");
    relayout_kernel<<<(unsigned)blocks_for(total, 256, 16), 256, 0, (cudaStream_t)stream>>>(
        T, M, N, layout_strides(src_layout, T, M, N), layout_strides(dst_layout, T, M, N), dst_layout,
        src_dev, dst_dev);
    return check_launch("relayout_kernel");
}

extern "C" int fvb_aos_to_soa(int dim, int p, int64_t T, int haloed, const double* aos_dev,
                              double* soa_dev, void* stream) {
    return aos_soa(dim, p, T, haloed, aos_dev, soa_dev, stream, 1);
}

extern "C" int fvb_soa_to_aos(int dim, int p, int64_t T, int haloed, const double* soa_dev,
                              double* aos_dev, void* stream) {
    return aos_soa(dim, p, T, haloed, soa_dev, aos_dev, stream, 0);
}

// ---------------------------------------------------------------------------
// microkernel probe + admissibility
// ---------------------------------------------------------------------------
template <int D, class R>
__device__ __forceinline__ void probe_one(const Euler<D>& eq, const double* q, int axis, double* f,
                                          double* lam) {
    constexpr int N = D + 2;
    R s[N], fl[N];
#pragma unroll
    for (int k = 0; k < N; ++k) s[k] = q[k];
    eq.flux(s, axis, fl);
    const R l = eq.max_eigenvalue(s, axis);
#pragma unroll
    for (int k = 0; k < N; ++k) f[k] = val(fl[k]);
    *lam = val(l);
}

// policy 0: IEEE double; policy 1: the kernels' XReal fast paths with the
// IEEE redo when a fast path leaves its range (what the fused kernels do).
template <int D>
__global__ void microkernel_probe_kernel(long long count, int axis, double gamma, int policy,
                                         const double* __restrict__ q, double* __restrict__ f,
                                         double* __restrict__ lam) {
    constexpr int N = D + 2;
    const Euler<D> eq{gamma};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        double fl[N], l, s[N];
#pragma unroll
        for (int k = 0; k < N; ++k) s[k] = q[i * N + k];
        if (policy == 1 && eq.fast_path_safe(s)) probe_one<D, XReal>(eq, s, axis, fl, &l);
        else probe_one<D, double>(eq, s, axis, fl, &l);
#pragma unroll
        for (int k = 0; k < N; ++k) f[i * N + k] = fl[k];
        lam[i] = l;
    }
}

extern "C" int fvb_eval_microkernels(int dim, int64_t count, int axis, double gamma, int policy,
                                     const double* q_dev, double* flux_dev, double* lambda_dev,
                                     void* stream) {
    if (dim != 2 && dim != 3) return fail(FVB_EINVAL, "dim must be 2 or 3, got %d", dim);
    if (axis < 0 || axis >= dim) return fail(FVB_EINVAL, "axis %d out of range for d=%d", axis, dim);
    if (policy != 0 && policy != 1) return fail(FVB_EINVAL, "policy must be 0 or 1, got %d", policy);
    if (count < 0) return fail(FVB_EINVAL, "negative count");
    if (count == 0) return FVB_OK;
    const unsigned grid = (unsigned)blocks_for(count, 256, 16);
    cudaStream_t st = (cudaStream_t)stream;
    if (dim == 2)
        microkernel_probe_kernel<2><<<grid, 256, 0, st>>>(count, axis, gamma, policy, q_dev, flux_dev, lambda_dev);
    else
        microkernel_probe_kernel<3><<<grid, 256, 0, st>>>(count, axis, gamma, policy, q_dev, flux_dev, lambda_dev);
    return check_launch("microkernel_probe_kernel");
}

// Raw fast paths: quotient a/b and sqrt(a) as XReal computes them, plus the
// range flags (bit 0: division left its fast path, bit 1: sqrt did).
__global__ void fastmath_probe_kernel(long long count, const double* __restrict__ a,
                                      const double* __restrict__ b, double* __restrict__ quot,
                                      double* __restrict__ root, int* __restrict__ flags) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        const double q = fast_div(a[i], b[i]);
        const double r = fast_sqrt(a[i]);
        quot[i] = q;
        root[i] = r;
        flags[i] = (div_fast_ok(a[i], b[i], q) ? 0 : 1) | (sqrt_fast_ok(a[i]) ? 0 : 2);
    }
}

extern "C" int fvb_probe_fastmath(int64_t count, const double* a_dev, const double* b_dev,
                                  double* quot_dev, double* root_dev, int32_t* flags_dev,
                                  void* stream) {
    if (count < 0) return fail(FVB_EINVAL, "negative count");
    if (count == 0) return FVB_OK;
    fastmath_probe_kernel<<<(unsigned)blocks_for(count, 256, 16), 256, 0, (cudaStream_t)stream>>>(
        count, a_dev, b_dev, quot_dev, root_dev, flags_dev);
    return check_launch("fastmath_probe_kernel");
}

// Check mode evaluates exactly the states the reference's step passes to
// pressure(..., check=True): the flux ranges of the input (cells with at
// most one halo coordinate -- corner halo cells are never read,
// microkernels.py:138, :153) and the interior output cells of the reduce
// (microkernels.py:190).
template <int D>
__global__ void admissible_kernel(long long T, int p, int haloed, double gamma, Lay lay,
                                  const double* __restrict__ q, const double* const* __restrict__ tab,
                                  unsigned long long* __restrict__ bad) {
    constexpr int N = D + 2;
    const Euler<D> eq{gamma};
    const int m = haloed ? p + 2 : p;
    const long long M = ipow_d(m, D);
    const long long total = T * M;
    unsigned long long local = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long patch = i / M;
        const int lin = (int)(i - patch * M);
        if (haloed) {
            int rest = lin, halo = 0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const int c = rest % m;
                rest /= m;
                halo += (c == 0 || c == m - 1) ? 1 : 0;
            }
            if (halo > 1) continue;
        }
        const double* base = tab != nullptr ? tab[patch] : q + patch * lay.p;
        double s[N];
#pragma unroll
        for (int k = 0; k < N; ++k) s[k] = base[k * lay.k + (long long)lin * lay.l];
        if (!(s[0] > 0.0) || !(eq.pressure(s) > 0.0)) ++local;
    }
    if (local) atomicAdd(bad, local);
}

extern "C" int fvb_check_admissible_ex(int dim, int p, int64_t T, int haloed, int layout, double gamma,
                                       const double* q_dev, const double* const* tab_dev,
                                       int64_t* bad_count_dev, void* stream) {
    int rc = validate_shape(dim, p, T);
    if (rc) return rc;
    if (layout != FVB_LAYOUT_AOS && layout != FVB_LAYOUT_SOA && layout != FVB_LAYOUT_AOSOA)
        return fail(FVB_EINVAL, "unknown layout %d", layout);
    if (tab_dev != nullptr) layout = FVB_LAYOUT_AOS;  // per-patch arrays are AoS
    else if (q_dev == nullptr) return fail(FVB_EINVAL, "null batch");
    cudaStream_t st = (cudaStream_t)stream;
    FVB_CUDA(cudaMemsetAsync(bad_count_dev, 0, sizeof(int64_t), st));
    const long long M = ipow_h(haloed ? p + 2 : p, dim), total = T * M;
    const Lay lay = layout_strides(layout, T, M, dim + 2);
    const unsigned grid = (unsigned)blocks_for(total, 256, 16);
    auto* bad = reinterpret_cast<unsigned long long*>(bad_count_dev);
    if (dim == 2) admissible_kernel<2><<<grid, 256, 0, st>>>(T, p, haloed, gamma, lay, q_dev, tab_dev, bad);
    else admissible_kernel<3><<<grid, 256, 0, st>>>(T, p, haloed, gamma, lay, q_dev, tab_dev, bad);
    return check_launch("admissible_kernel");
}

extern "C" int fvb_check_admissible(int dim, int p, int64_t T, int haloed, double gamma,
                                    const double* q_dev, int64_t* bad_count_dev, void* stream) {
    return fvb_check_admissible_ex(dim, p, T, haloed, FVB_LAYOUT_SOA, gamma, q_dev, nullptr, bad_count_dev,
                                   stream);
}

extern "C" double fvb_admissible_dt(double lambda, double h, double cfl) { return cfl * h / lambda; }

// The same expression on the device, from the device eigenvalue (a multi-step
// run then never waits for the host; bit-identical to fvb_admissible_dt).
__global__ void admissible_dt_kernel(const double* lam, double h, double cfl, double* dt) {
    *dt = __ddiv_rn(__dmul_rn(cfl, h), *lam);
}

extern "C" int fvb_admissible_dt_dev(const double* lam_dev, double h, double cfl, double* dt_dev,
                                     void* stream) {
    if (lam_dev == nullptr || dt_dev == nullptr) return fail(FVB_EINVAL, "null pointer");
    admissible_dt_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(lam_dev, h, cfl, dt_dev);
    return check_launch("admissible_dt_kernel");
}

// RCP64H scaling probe (test support for XScaled in realx.cuh): for every
// high-word mantissa pattern m (2^20 of them) and every biased exponent e in
// [e_lo, e_hi], x = (e, m, low word = hash) must satisfy
// fast_recip(2x) == 0.5 * fast_recip(x) bit for bit.  Counts violations.
__global__ void rcp_scaling_kernel(int e_lo, int e_hi, unsigned long long* bad) {
    const long long total = (long long)(e_hi - e_lo + 1) << 20;
    unsigned long long local = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int e = e_lo + (int)(i >> 20);
        const int m = (int)(i & 0xfffff);
        const unsigned lo = (unsigned)(i * 2654435761ull) ^ 0x9e3779b9u;
        const double x = __hiloint2double((e << 20) | m, (int)lo);
        const double r2 = fast_recip(__dmul_rn(2.0, x));
        const double r1 = 0.5 * fast_recip(x);
        if (__double_as_longlong(r2) != __double_as_longlong(r1)) ++local;
    }
    if (local) atomicAdd(bad, local);
}

extern "C" int fvb_probe_rcp_scaling(int e_lo, int e_hi, int64_t* mismatches_dev, void* stream) {
    if (e_lo < 1 || e_hi > 2045 || e_lo > e_hi) return fail(FVB_EINVAL, "exponent range [%d, %d]", e_lo, e_hi);
    cudaStream_t st = (cudaStream_t)stream;
    FVB_CUDA(cudaMemsetAsync(mismatches_dev, 0, sizeof(int64_t), st));
    rcp_scaling_kernel<<<(unsigned)blocks_for((long long)(e_hi - e_lo + 1) << 20, 256, 16), 256, 0, st>>>(
        e_lo, e_hi, reinterpret_cast<unsigned long long*>(mismatches_dev));
    return check_launch("rcp_scaling_kernel");
}

// ---------------------------------------------------------------------------
// halo refresh for a Cartesian grid of patches (multi-step driver, f2 row)
// ---------------------------------------------------------------------------
// Patches form a px x py (x pz) grid, patch index ix + px*(iy + py*iz).  For
// every haloed cell of every patch, copy the interior cell it overlaps: its
// own interior or a neighbour's (periodic wrap).  Input: the interior SoA
// output of the previous step; output: the haloed SoA input of the next.
template <int D>
__global__ void refresh_halos_kernel(int p, int px, int py, int pz, const double* __restrict__ src,
                                     double* __restrict__ dst) {
    constexpr int N = D + 2;
    const int m = p + 2;
    const long long M = ipow_d(m, D), Mi = ipow_d(p, D);
    const long long T = (long long)px * py * pz;
    const long long total = T * M;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long patch = i / M;
        int lin = (int)(i - patch * M);
        int pc[3] = {(int)(patch % px), (int)((patch / px) % py), (int)(patch / ((long long)px * py))};
        const int pn[3] = {px, py, pz};
        int cell[3] = {0, 0, 0};
#pragma unroll
        for (int k = 0; k < D; ++k) {
            int c = lin % m - 1;  // haloed coordinate -1..p
            lin /= m;
            if (c < 0) c += p, pc[k] = (pc[k] + pn[k] - 1) % pn[k];
            else if (c >= p) c -= p, pc[k] = (pc[k] + 1) % pn[k];
            cell[k] = c;
        }
        const long long sp = pc[0] + (long long)px * (pc[1] + (long long)py * pc[2]);
        long long li = 0;
#pragma unroll
        for (int k = D - 1; k >= 0; --k) li = li * p + cell[k];
#pragma unroll
        for (int k = 0; k < N; ++k) dst[k * total + i] = __ldg(src + k * T * Mi + sp * Mi + li);
    }
}

extern "C" int fvb_refresh_halos(int dim, int p, int px, int py, int pz, const double* interior_dev,
                                 double* haloed_dev, void* stream) {
    if (px < 1 || py < 1 || pz < 1 || (dim == 2 && pz != 1))
        return fail(FVB_EINVAL, "bad patch grid %d x %d x %d for d=%d", px, py, pz, dim);
    int rc = validate_shape(dim, p, (int64_t)px * py * pz);
    if (rc) return rc;
    const long long total = (long long)px * py * pz * ipow_h(p + 2, dim);
    const unsigned grid = (unsigned)blocks_for(total, 256, 16);
    cudaStream_t st = (cudaStream_t)stream;
    if (dim == 2) refresh_halos_kernel<2><<<grid, 256, 0, st>>>(p, px, py, pz, interior_dev, haloed_dev);
    else refresh_halos_kernel<3><<<grid, 256, 0, st>>>(p, px, py, pz, interior_dev, haloed_dev);
    return check_launch("refresh_halos_kernel");
}
