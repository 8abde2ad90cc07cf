// rr_k_pair_chain.cu — march-kernel instantiations for general diffeo chains
// (affine / twist / bend / local bump stages, RK4) on the ray-pair kernel:
// march2_kernel<kDiffeoChain> with and without meshes (see rr_march.cuh,
// accel_diffeo_x2).
#include "rr_march.cuh"

namespace rr {

cudaError_t launch_family_pair_chain(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                     const char** name) {
    if (P.n_meshes > 0) {
        *name = "march2_kernel<diffeo,mesh>";
        return launch_variant2<kDiffeoChain, 0, true>(P, L, s, sms);
    }
    *name = "march2_kernel<diffeo>";
    return launch_variant2<kDiffeoChain, 0, false>(P, L, s, sms);
}

} // namespace rr
