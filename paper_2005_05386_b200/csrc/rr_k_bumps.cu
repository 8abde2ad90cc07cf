// rr_k_bumps.cu — march-kernel instantiations for Gaussian-bump graph metrics on the one-ray kernel (Euler, rk23, meshes) (see rr_march.cuh).
#include "rr_march.cuh"

namespace rr {
namespace {

template <int SCHEME, bool MESH>
cudaError_t bumps_scheme(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                         const char** name) {
    if constexpr (!MESH && SCHEME != 2) {   // mesh / rk23 scenes use 16/32 slots only
        if (P.nb_slot <= 4) {
            *name = "march_kernel<bumps4>";
            return launch_variant<kBumps, 4, SCHEME, MESH>(P, L, s, sms);
        }
        if (P.nb_slot <= 8) {
            *name = "march_kernel<bumps8>";
            return launch_variant<kBumps, 8, SCHEME, MESH>(P, L, s, sms);
        }
    }
    if (P.nb_slot <= 16) {
        *name = MESH ? "march_kernel<bumps16,mesh>" : "march_kernel<bumps16>";
        return launch_variant<kBumps, 16, SCHEME, MESH>(P, L, s, sms);
    }
    *name = MESH ? "march_kernel<bumps32,mesh>" : "march_kernel<bumps32>";
    return launch_variant<kBumps, 32, SCHEME, MESH>(P, L, s, sms);
}

template <bool MESH>
cudaError_t bumps_mesh(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms, const char** name) {
    if (P.scheme == 2) return bumps_scheme<2, MESH>(P, L, s, sms, name);
    return P.scheme == 0 ? bumps_scheme<0, MESH>(P, L, s, sms, name)
                         : bumps_scheme<1, MESH>(P, L, s, sms, name);
}

} // namespace

cudaError_t launch_family_bumps(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                const char** name) {
    return P.n_meshes > 0 ? bumps_mesh<true>(P, L, s, sms, name) : bumps_mesh<false>(P, L, s, sms, name);
}

} // namespace rr
