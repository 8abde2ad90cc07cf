// rr_k_flat.cu — march-kernel instantiations for the Euclidean metric and general graph fields (polynomials, > 32 Gaussians) (see rr_march.cuh).
#include "rr_march.cuh"

namespace rr {
namespace {

template <int KIND, bool MESH>
cudaError_t fam_mesh(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms) {
    if (P.scheme == 2) return launch_variant<KIND, 0, 2, MESH>(P, L, s, sms);
    return P.scheme == 0 ? launch_variant<KIND, 0, 0, MESH>(P, L, s, sms)
                         : launch_variant<KIND, 0, 1, MESH>(P, L, s, sms);
}

} // namespace

cudaError_t launch_family_euclid(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                 const char** name) {
    *name = P.n_meshes > 0 ? "march_kernel<euclid,mesh>" : "march_kernel<euclid>";
    return P.n_meshes > 0 ? fam_mesh<kEuclid, true>(P, L, s, sms) : fam_mesh<kEuclid, false>(P, L, s, sms);
}

cudaError_t launch_family_graph(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                const char** name) {
    *name = P.n_meshes > 0 ? "march_kernel<graph,mesh>" : "march_kernel<graph>";
    return P.n_meshes > 0 ? fam_mesh<kGraphGeneral, true>(P, L, s, sms)
                          : fam_mesh<kGraphGeneral, false>(P, L, s, sms);
}

} // namespace rr
