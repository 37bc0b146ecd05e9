// cascade.cu -- launchers of the per-step kernels (cascade.cuh): the cascade
// flavour enqueues them in stream order; the graph flavour (fvb.cu) adds them
// as CUDA Graph nodes via cascade_fns().
#include "cascade.cuh"
#include "host.h"

namespace fvb {

CascadeFns cascade_fns(int dim) {
    if (dim == 2)
        return {(void*)cascade_copy_kernel<2>, (void*)cascade_flux_kernel<2, false>,
                (void*)cascade_flux_kernel<2, true>, (void*)cascade_acc_kernel<2>,
                (void*)cascade_reduce_kernel<2, kReduceThreads>};
    return {(void*)cascade_copy_kernel<3>, (void*)cascade_flux_kernel<3, false>,
            (void*)cascade_flux_kernel<3, true>, (void*)cascade_acc_kernel<3>,
            (void*)cascade_reduce_kernel<3, kReduceThreads>};
}

int launch_cascade(int d, const CascadeArgs& ca, bool reduce, cudaStream_t st) {
    const StepArgs& a = ca.s;
    const long long span = a.t1 - a.t0;
    const long long Mi = ipow_h(a.p, d), R = (a.p + 2) * ipow_h(a.p, d - 1);
    const unsigned gi = (unsigned)blocks_for(span * Mi, kEltThreads, 16);
    const unsigned gr = (unsigned)blocks_for(span * R, kEltThreads, 16);
    if (d == 2) {
        cascade_copy_kernel<2><<<gi, kEltThreads, 0, st>>>(a);
        for (int ax = 0; ax < 2; ++ax) cascade_flux_kernel<2, false><<<gr, kEltThreads, 0, st>>>(ca, ax);
        for (int ax = 0; ax < 2; ++ax) cascade_flux_kernel<2, true><<<gr, kEltThreads, 0, st>>>(ca, ax);
        for (int ax = 0; ax < 2; ++ax) cascade_acc_kernel<2><<<gi, kEltThreads, 0, st>>>(ca, ax);
        if (reduce) cascade_reduce_kernel<2, kReduceThreads><<<gi, kReduceThreads, 0, st>>>(a);
    } else {
        cascade_copy_kernel<3><<<gi, kEltThreads, 0, st>>>(a);
        for (int ax = 0; ax < 3; ++ax) cascade_flux_kernel<3, false><<<gr, kEltThreads, 0, st>>>(ca, ax);
        for (int ax = 0; ax < 3; ++ax) cascade_flux_kernel<3, true><<<gr, kEltThreads, 0, st>>>(ca, ax);
        for (int ax = 0; ax < 3; ++ax) cascade_acc_kernel<3><<<gi, kEltThreads, 0, st>>>(ca, ax);
        if (reduce) cascade_reduce_kernel<3, kReduceThreads><<<gi, kReduceThreads, 0, st>>>(a);
    }
    return check_launch("cascade kernels");
}

}  // namespace fvb
