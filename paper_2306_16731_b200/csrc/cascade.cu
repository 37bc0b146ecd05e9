// cascade.cu -- launchers of the per-step kernels (cascade.cuh): the cascade
// flavour enqueues them in stream order; the graph flavour (fvb.cu) adds them
// as CUDA Graph nodes via cascade_fns().
#include "cascade.cuh"
#include "host.h"

namespace fvb {

namespace {

template <class Eq>
CascadeFns fns_of() {
    return {(void*)cascade_copy_kernel<Eq>, (void*)cascade_flux_kernel<Eq, false>,
            (void*)cascade_flux_kernel<Eq, true>, (void*)cascade_acc_kernel<Eq>,
            (void*)cascade_reduce_kernel<Eq, kReduceThreads>};
}

template <class Eq>
int launch(const CascadeArgs& ca, bool reduce, cudaStream_t st) {
    constexpr int d = Eq::kDim;
    const StepArgs& a = ca.s;
    const long long span = a.t1 - a.t0;
    const long long Mi = ipow_h(a.p, d), R = (a.p + 2) * ipow_h(a.p, d - 1);
    const unsigned gi = (unsigned)blocks_for(span * Mi, kEltThreads, 16);
    const unsigned gr = (unsigned)blocks_for(span * R, kEltThreads, 16);
    cascade_copy_kernel<Eq><<<gi, kEltThreads, 0, st>>>(a);
    for (int ax = 0; ax < d; ++ax) cascade_flux_kernel<Eq, false><<<gr, kEltThreads, 0, st>>>(ca, ax);
    for (int ax = 0; ax < d; ++ax) cascade_flux_kernel<Eq, true><<<gr, kEltThreads, 0, st>>>(ca, ax);
    for (int ax = 0; ax < d; ++ax) cascade_acc_kernel<Eq><<<gi, kEltThreads, 0, st>>>(ca, ax);
    if (reduce) cascade_reduce_kernel<Eq, kReduceThreads><<<gi, kReduceThreads, 0, st>>>(a);
    return check_launch("cascade kernels");
}

}  // namespace

CascadeFns cascade_fns(int dim, int physics) {
    auto get = [](auto tag) { return fns_of<typename decltype(tag)::type>(); };
    return dim == 2 ? with_physics<2>(physics, get) : with_physics<3>(physics, get);
}

int launch_cascade(int d, const CascadeArgs& ca, bool reduce, cudaStream_t st) {
    auto go = [&](auto tag) { return launch<typename decltype(tag)::type>(ca, reduce, st); };
    return d == 2 ? with_physics<2>(ca.s.physics, go) : with_physics<3>(ca.s.physics, go);
}

}  // namespace fvb
