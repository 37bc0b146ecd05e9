// physics.cuh -- the domain-policy contract every step kernel is templated on.
//
// The reference's microkernels are user code the executors call but never
// alter (pkg/src/patchbench/equations.py:11-12, :60-107; microkernels.py:10-13).
// Here a "physics" is a policy struct; the kernels (fused 2D pencil, fused 3D
// plane walks, generic, cascade / graph) take it as a template parameter and
// call only these members:
//
//   required
//     static constexpr int kDim;        // d
//     static constexpr int kUnknowns;   // N (the state vector length)
//     explicit Eq(double gamma);        // from the run parameters (EulerParameters)
//     void   flux(const double (&q)[N], int axis, double (&f)[N]) const;
//     double max_eigenvalue(const double (&q)[N], int axis) const;
//
//   optional hooks (detected at compile time, never required)
//     fast_path_safe(const XReal (&q)[N])   + flux / max_eigenvalue templated
//         on the scalar type: the fused kernels first evaluate certified
//         states with XReal (realx.cuh: CUDA's fp64 '/' and sqrt fast paths
//         written out) and redo a patch group in IEEE double when a state is
//         not certified.  Without it every state is evaluated in IEEE double.
//     lambda_below(const double (&q)[N], double tau_lo): a sufficient test
//         that max_n max_eigenvalue(q, n) < tau; enables the filtered
//         eigenvalue reduction.  Without it the reduction is exhaustive
//         (every finished cell's max_eigenvalue, executors.py:140-211).
//
// Either way the results are the reference's bits: the hooks only choose
// cheaper instruction sequences for the same IEEE values.
//
// Policies shipped (selected at run time with fvb_set_physics, include/fvb.h):
//   FVB_PHYSICS_EULER        Euler<D>      (euler.cuh: both hooks)
//   FVB_PHYSICS_EULER_PLAIN  EulerPlain<D> (below: the reference's three
//                            functions only, plain double -- what a user
//                            writes; it exercises the hook-free paths)
// Adding a policy: a struct with the members above + one line in
// FVB_PHYSICS_LIST (host.h) -- no kernel edits.
#pragma once

#include <type_traits>
#include <utility>

#include "euler.cuh"
#include "realx.cuh"

namespace fvb {

template <class Eq, class = void>
struct has_fast_path : std::false_type {};
template <class Eq>
struct has_fast_path<Eq, std::void_t<decltype(std::declval<const Eq&>().fast_path_safe(
                             std::declval<const XReal (&)[Eq::kUnknowns]>()))>> : std::true_type {};
template <class Eq>
constexpr bool kHasFastPath = has_fast_path<Eq>::value;

template <class Eq, class = void>
struct has_lambda_below : std::false_type {};
template <class Eq>
struct has_lambda_below<Eq, std::void_t<decltype(std::declval<const Eq&>().lambda_below(
                                std::declval<const double (&)[Eq::kUnknowns]>(), 0.0))>> : std::true_type {};
template <class Eq>
constexpr bool kHasLambdaBelow = has_lambda_below<Eq>::value;

// The compressible Euler closure exactly as the reference's user code states
// it (equations.py:60-107), plain IEEE double, no hooks.
template <int D>
struct EulerPlain {
    static constexpr int kDim = D;
    static constexpr int kUnknowns = D + 2;
    double gamma;
    __host__ __device__ explicit EulerPlain(double g) : gamma(g) {}

    // equations.py:60-74
    __device__ __forceinline__ double pressure(const double (&q)[D + 2]) const {
        double ke = q[1] * q[1] + q[2] * q[2];
        if (D == 3) ke = ke + q[3] * q[3];
        return (gamma - 1.0) * (q[D + 1] - ke / (2.0 * q[0]));
    }
    // equations.py:77-95
    __device__ __forceinline__ void flux(const double (&q)[D + 2], int axis, double (&f)[D + 2]) const {
        const double p = pressure(q);
        const double un = q[1 + axis] / q[0];
        f[0] = q[1 + axis];
#pragma unroll
        for (int i = 0; i < D; ++i) f[1 + i] = (i == axis) ? q[1 + i] * un + p : q[1 + i] * un;
        f[D + 1] = un * (q[D + 1] + p);
    }
    // equations.py:98-107
    __device__ __forceinline__ double max_eigenvalue(const double (&q)[D + 2], int axis) const {
        const double p = pressure(q);
        return fabs(q[1 + axis] / q[0]) + sqrt(gamma * p / q[0]);
    }
};

static_assert(kHasFastPath<Euler<2>> && kHasLambdaBelow<Euler<3>>, "Euler carries both hooks");
static_assert(!kHasFastPath<EulerPlain<2>> && !kHasLambdaBelow<EulerPlain<3>>, "EulerPlain carries none");

}  // namespace fvb
