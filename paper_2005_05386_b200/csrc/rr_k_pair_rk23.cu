// rr_k_pair_rk23.cu — march-kernel instantiations for Gaussian-bump frames
// with the adaptive rk23 scheme (EXTENSION) on the ray-pair kernel
// (march2_kernel<kBumpsRk23>, march_pair_rk23 in rr_march.cuh).
#include "rr_march.cuh"

namespace rr {

cudaError_t launch_family_pair_rk23(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                    const char** name) {
    if (P.nb_slot <= 16) {
        *name = "march2_kernel<bumps16,rk23>";
        return launch_variant2<kBumpsRk23, 16, false>(P, L, s, sms);
    }
    *name = "march2_kernel<bumps32,rk23>";
    return launch_variant2<kBumpsRk23, 32, false>(P, L, s, sms);
}

} // namespace rr
