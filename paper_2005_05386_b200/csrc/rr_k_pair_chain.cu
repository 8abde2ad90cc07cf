// rr_k_pair_chain.cu — march-kernel instantiations for general diffeo chains
// (affine / twist / bend / local bump stages, RK4) on the ray-pair kernel:
// march2_kernel<kDiffeoChain, SIG> with and without meshes (see rr_march.cuh,
// accel_diffeo_x2).  SIG 0 folds any chain with a run-time loop over the
// stage kinds; the BASELINE configs[3] chain (twist o bend, in either order)
// gets a fold specialised at compile time.
#include "rr_march.cuh"

namespace rr {

namespace {

template <int SIG>
cudaError_t launch_chain(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms) {
    return P.n_meshes > 0 ? launch_variant2<kDiffeoChain, SIG, true>(P, L, s, sms)
                          : launch_variant2<kDiffeoChain, SIG, false>(P, L, s, sms);
}

}  // namespace

cudaError_t launch_family_pair_chain(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                     const char** name) {
    *name = P.n_meshes > 0 ? "march2_kernel<diffeo,mesh>" : "march2_kernel<diffeo>";
#if RR_CHAIN_STATIC
    if (P.n_stages == 2) {
        const int k0 = P.stages[0].kind, k1 = P.stages[1].kind;
        if (k0 == kStageBend && k1 == kStageTwist)
            return launch_chain<chain_sig2(kStageBend, kStageTwist)>(P, L, s, sms);
        if (k0 == kStageTwist && k1 == kStageBend)
            return launch_chain<chain_sig2(kStageTwist, kStageBend)>(P, L, s, sms);
    }
#endif
    return launch_chain<0>(P, L, s, sms);
}

} // namespace rr
