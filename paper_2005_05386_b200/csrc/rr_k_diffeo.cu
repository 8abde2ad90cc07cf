// rr_k_diffeo.cu — march-kernel instantiations for diffeomorphism pull-back metrics (twist / bend / bump / affine chains) (see rr_march.cuh).
#include "rr_march.cuh"

namespace rr {
namespace {

template <bool MESH>
cudaError_t fam_mesh(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms, const char** name) {
    *name = MESH ? "march_kernel<diffeo,mesh>" : "march_kernel<diffeo>";
    if (P.scheme == 2) return launch_variant<kDiffeo, 0, 2, MESH>(P, L, s, sms);
#if RR_TWIST_ONE_STATIC
    // the single twist with meshes (C4): a variant without the general fold
    if (MESH && P.scheme == 1 && P.n_stages == 1 && P.stages[0].kind == kStageTwist)
        return launch_variant<kDiffeo, 1, 1, MESH>(P, L, s, sms);
#endif
    return P.scheme == 0 ? launch_variant<kDiffeo, 0, 0, MESH>(P, L, s, sms)
                         : launch_variant<kDiffeo, 0, 1, MESH>(P, L, s, sms);
}

} // namespace

cudaError_t launch_family_diffeo(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                 const char** name) {
    return P.n_meshes > 0 ? fam_mesh<true>(P, L, s, sms, name) : fam_mesh<false>(P, L, s, sms, name);
}

} // namespace rr
