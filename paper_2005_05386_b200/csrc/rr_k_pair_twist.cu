// rr_k_pair_twist.cu — march-kernel instantiations for the single-twist
// pull-back metric (C4) on the ray-pair kernel: march2_kernel<kDiffeo> with
// and without meshes (see rr_march.cuh).
#include "rr_march.cuh"

namespace rr {

cudaError_t launch_family_pair_twist(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                     const char** name) {
    if (P.n_meshes > 0) {
        *name = "march2_kernel<twist,mesh>";
        return launch_variant2<kDiffeo, 0, true>(P, L, s, sms);
    }
    *name = "march2_kernel<twist>";
    return launch_variant2<kDiffeo, 0, false>(P, L, s, sms);
}

} // namespace rr
