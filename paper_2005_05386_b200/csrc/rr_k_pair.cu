// rr_k_pair.cu — march-kernel instantiations for Gaussian-bump RK4 frames and batches: the ray-pair kernel march2_kernel (see rr_march.cuh).
#include "rr_march.cuh"

namespace rr {
namespace {

template <int NB>
cudaError_t pair_nb(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms, const char** name,
                    const char* label) {
    *name = label;
    return launch_variant2<kBumps, NB, false>(P, L, s, sms);
}

} // namespace

cudaError_t launch_family_pair(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                               const char** name) {
    if (P.nb_slot <= 4) return pair_nb<4>(P, L, s, sms, name, "march2_kernel<bumps4>");
    if (P.nb_slot <= 8) return pair_nb<8>(P, L, s, sms, name, "march2_kernel<bumps8>");
    if (P.nb_slot <= 16) return pair_nb<16>(P, L, s, sms, name, "march2_kernel<bumps16>");
    return pair_nb<32>(P, L, s, sms, name, "march2_kernel<bumps32>");
}

} // namespace rr
