// Compile-only check of the physics contract (csrc/physics.cuh): a policy
// with a DIFFERENT unknown count -- 2D / 3D Euler carrying a passive tracer
// (N = d + 3), stated as a user would: the three functions, plain double,
// no hooks -- instantiates every fused and cascade kernel template.  The
// host batch format stays the reference's (N = d + 2), so the library does
// not dispatch to it; tests/test_physics_compile.py only builds this file.
#include "../../paper_2306_16731_b200/csrc/cascade.cuh"
#include "../../paper_2306_16731_b200/csrc/fused2d_tile.cuh"
#include "../../paper_2306_16731_b200/csrc/fused2d_tma.cuh"
#include "../../paper_2306_16731_b200/csrc/fused3d_warp.cuh"
#include "../../paper_2306_16731_b200/csrc/fused_generic.cuh"

namespace user {

template <int D>
struct EulerTracer {
    static constexpr int kDim = D;
    static constexpr int kUnknowns = D + 3;  // rho, rho*u_0..u_{d-1}, E, rho*phi
    double gamma;
    __host__ __device__ explicit EulerTracer(double g) : gamma(g) {}
    __device__ double pressure(const double (&q)[D + 3]) const {
        double ke = q[1] * q[1] + q[2] * q[2];
        if (D == 3) ke = ke + q[3] * q[3];
        return (gamma - 1.0) * (q[D + 1] - ke / (2.0 * q[0]));
    }
    __device__ void flux(const double (&q)[D + 3], int axis, double (&f)[D + 3]) const {
        const double p = pressure(q);
        const double un = q[1 + axis] / q[0];
        f[0] = q[1 + axis];
        for (int i = 0; i < D; ++i) f[1 + i] = (i == axis) ? q[1 + i] * un + p : q[1 + i] * un;
        f[D + 1] = un * (q[D + 1] + p);
        f[D + 2] = q[D + 2] * un;  // the tracer is advected
    }
    __device__ double max_eigenvalue(const double (&q)[D + 3], int axis) const {
        const double p = pressure(q);
        return fabs(q[1 + axis] / q[0]) + sqrt(gamma * p / q[0]);
    }
};

}  // namespace user

namespace fvb {
// one instantiation of every kernel family with the N = d + 3 policy
template __global__ void fused2d_pencil_kernel<user::EulerTracer<2>, 16, 1, 1, kReduceAll, 12, 3, 1>(StepArgs);
template __global__ void fused2d_pencil_tma_kernel<user::EulerTracer<2>, 16, kReduceAll, 12, 3, 2, false>(
    StepArgs, const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void fused2d_tile_kernel<user::EulerTracer<2>, 3, kReduceAll, 4, 1, true>(StepArgs);
template __global__ void fused3d_warp_kernel<user::EulerTracer<3>, 8, 2, kReduceAll, 8, 1>(
    StepArgs, const __grid_constant__ CUtensorMap, int);
template __global__ void fused3d_slab_kernel<user::EulerTracer<3>, 4, 1, 4, kReduceAll, 6, 1>(StepArgs);
template __global__ void fused_generic_kernel<user::EulerTracer<3>, 256, true>(StepArgs);
template __global__ void cascade_flux_kernel<user::EulerTracer<2>, false>(CascadeArgs, int);
template __global__ void cascade_acc_kernel<user::EulerTracer<3>>(CascadeArgs, int);
template __global__ void cascade_reduce_kernel<user::EulerTracer<3>, 256>(StepArgs);
static_assert(!kHasFastPath<user::EulerTracer<2>> && !kHasLambdaBelow<user::EulerTracer<3>>, "hook-free");
}  // namespace fvb
