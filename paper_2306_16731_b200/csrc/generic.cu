// generic.cu -- launcher of the fused shared-memory kernel (fused_generic.cuh):
// 3D patches and 2D patches the pencil kernel does not cover.
#include "fused_generic.cuh"
#include "host.h"

namespace fvb {
namespace {

constexpr int kGenericThreads = 256;

template <class Eq, bool R>
int launch(const StepArgs& a, cudaStream_t st) {
    constexpr int D = Eq::kDim;
    auto kern = fused_generic_kernel<Eq, kGenericThreads, R>;
    const long long smem = generic_smem_bytes(D, a.p);
    if (smem > smem_optin())
        return fail(FVB_ELIMIT,
                    "(p+2)^d staging for d=%d p=%d needs %lld B shared memory > %d B per CTA; "
                    "use the cascade or graph flavour",
                    D, a.p, smem, smem_optin());
    static PerDevice configured_dev;
    int& configured = configured_dev();
    if (!configured) {
        FVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin()));
        configured = 1;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGenericThreads, (size_t)smem);
    if (occ <= 0) occ = 1;
    long long blocks = a.t1 - a.t0;
    const long long cap = (long long)sm_count() * occ;
    if (blocks > cap) blocks = cap;
    kern<<<(unsigned)blocks, kGenericThreads, (size_t)smem, st>>>(a);
    return check_launch("fused_generic_kernel");
}

}  // namespace

long long generic_smem_bytes(int dim, int p) { return generic_smem_doubles(dim, p) * 8; }

int launch_generic(int dim, const StepArgs& a, bool reduce, cudaStream_t st) {
    auto go = [&](auto tag) {
        using Eq = typename decltype(tag)::type;
        return reduce ? launch<Eq, true>(a, st) : launch<Eq, false>(a, st);
    };
    return dim == 2 ? with_physics<2>(a.physics, go) : with_physics<3>(a.physics, go);
}

}  // namespace fvb
