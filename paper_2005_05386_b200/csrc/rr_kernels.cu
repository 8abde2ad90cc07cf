// rr_kernels.cu — launch dispatch and the small kernels of the B200 geodesic
// tracer (sm_100a): culling-grid build, detile, FFMA probe, geodesic export
// (trace) and flow_accel points.  The march kernels are instantiated per
// metric family in rr_k_pair.cu (ray-pair Gaussian-bump RK4), rr_k_bumps.cu,
// rr_k_diffeo.cu and rr_k_flat.cu (Euclidean + general graph fields).
#include "rr_march.cuh"

#include <cub/device/device_radix_sort.cuh>

namespace rr {
namespace {

// ---------------------------------------------------------------------------
// Culling grid build on the device (per scene upload, e.g. every animation
// frame).  Cell c gets bit slot(j) when bump j's R-sigma ellipsoid reaches the
// cell box dilated by `dil` (nearest point of the box to the centre, in sigma
// units; border cells extend to infinity because lookups clamp).  FP64, with
// the record's 1/sigma (a multiply instead of the divide: 1.38 -> 0.92 ms at
// 256^3, 0.59 -> 0.39 ms at 192^3 under ncu).
__global__ void cull_mask_kernel(const double* __restrict__ g, int n, int G, double lo0, double lo1,
                                 double lo2, double c0, double c1, double c2, double R2, double dil,
                                 uint32_t* __restrict__ masks) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= G * G * G) return;
    const int ix = idx % G, iy = (idx / G) % G, iz = idx / (G * G);
    const int id[3] = {ix, iy, iz};
    const double lo[3] = {lo0, lo1, lo2}, cell[3] = {c0, c1, c2};
    uint32_t m = 0;
    for (int j = 0; j < n; ++j) {
        const double* b = g + 8 * j;   // cx, cy, cz, 1/sx, 1/sy, 1/sz, slot, R_j^2
        double u2 = 0.0;
        for (int k = 0; k < 3; ++k) {
            const double a = id[k] == 0 ? -1e30 : lo[k] + id[k] * cell[k] - dil;
            const double e = id[k] == G - 1 ? 1e30 : lo[k] + (id[k] + 1) * cell[k] + dil;
            const double nr = fmin(fmax(b[k], a), e);
            const double u = (nr - b[k]) * b[3 + k];
            u2 += u * u;
        }
        if (u2 < fmin(R2, b[7])) m |= 1u << (int)b[6];
    }
    masks[idx] = m;
}

// One separable pass of the Chebyshev (L-inf) distance transform along axis
// `ax`: out(x) = min_y max(|x - y|, in(y)) over the grid line through x.
// Pass 0 reads the masks (0 where non-empty, infinity elsewhere).  One CTA
// per grid line: the line is staged in shared memory once and every thread
// scans it for its own x (an O(G) scan per cell, no global re-reads; the
// first build read each line G times from global memory, 0.6 ms per pass at
// G = 128).
__global__ void cheb_pass_kernel(const uint32_t* __restrict__ masks, const uint16_t* __restrict__ in,
                                 uint16_t* __restrict__ out, uint8_t* __restrict__ out8, int G, int ax) {
    extern __shared__ int line_v[];
    const int line = blockIdx.x;
    const int a = line % G, b = line / G;
    int stride, base;
    if (ax == 0) { stride = 1; base = (b * G + a) * G; }
    else if (ax == 1) { stride = G; base = b * G * G + a; }
    else { stride = G * G; base = b * G + a; }
    for (int y = threadIdx.x; y < G; y += blockDim.x)
        line_v[y] = masks ? (masks[base + y * stride] ? 0 : 0x7fff) : in[base + y * stride];
    __syncthreads();
    for (int x = threadIdx.x; x < G; x += blockDim.x) {
        int best = line_v[x];
        for (int y = 0; y < G; ++y) best = min(best, max(abs(x - y), line_v[y]));
        if (out8) out8[base + x * stride] = (uint8_t)min(best, 255);
        else out[base + x * stride] = (uint16_t)best;
    }
}

__global__ void detile_kernel(const uint8_t* __restrict__ g, int width, int height, int tw, int th,
                              int n_shards, int max_k, int tiles_x, uint8_t* __restrict__ rgb) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x;
    const int py = blockIdx.y;
    if (px >= width) return;
    const int tile = (py / th) * tiles_x + px / tw;
    const int shard = tile % n_shards, k = tile / n_shards;
    const size_t src = 3 * (((size_t)shard * max_k + k) * tw * th + (size_t)(py % th) * tw + px % tw);
    const size_t dst = 3 * ((size_t)py * width + px);
    rgb[dst] = g[src];
    rgb[dst + 1] = g[src + 1];
    rgb[dst + 2] = g[src + 2];
}

// Mesh free-distance grid (per scene upload): cell c gets
// floor(max(0, d(centre, nearest leaf box) - half diagonal) / q), a lower
// bound of the distance from any point of the cell to any triangle (every
// triangle lies in a leaf box), saturating at 255 q.
__global__ void mesh_dist_kernel(const float4* __restrict__ nodes, int G, float lo0, float lo1,
                                 float lo2, float c0, float c1, float c2, float q,
                                 uint8_t* __restrict__ out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= G * G * G) return;
    const int ix = idx % G, iy = (idx / G) % G, iz = idx / (G * G);
    const F3 centre = f3(lo0 + (ix + 0.5f) * c0, lo1 + (iy + 0.5f) * c1, lo2 + (iz + 0.5f) * c2);
    const float half_diag = 0.5f * sqrtf(c0 * c0 + c1 * c1 + c2 * c2);
    DevMesh M{};
    M.nodes = nodes;
    const float d = mesh_free(M, centre, 255.f * q + half_diag + q);
    // rounding margin of the FP32 distance: 1e-5 relative + 1e-5 absolute
    const float lb = fmaxf(0.f, d - half_diag - fmaf(1e-5f, d, 1e-5f));
    out[idx] = (uint8_t)fminf(255.f, floorf(lb / q));
}

__global__ void probe_kernel(uint8_t* p, uint8_t v) {
    *p = v;
    __threadfence_system();
}

// FFMA throughput probe: 8 independent FMA chains per thread, imm-free.
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678f) out[0] = s;   // keep the chains alive
}


// ---------------------------------------------------------------------------
// Off the render path (geodesic export + device verify): one thread per
// geodesic.  trace_geodesic (integrate.cpp:40-54): states[0] = start, one
// state per step, stop after the state that left the bounds (when asked) or
// at the first step whose metric evaluation failed (fail = step index).
// Positions carry the same compensated sum as the march.
template <int KIND, int NB, int SCHEME>
__global__ void __launch_bounds__(128) trace_kernel(const __grid_constant__ DevParams P,
                                                    const double* __restrict__ starts, int n,
                                                    float h, int max_steps, int use_bounds,
                                                    double* __restrict__ states,
                                                    int* __restrict__ counts, int* __restrict__ fail) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const double* s0 = starts + 6 * (size_t)r;
    double* out = states + (size_t)r * (size_t)(max_steps + 1) * 6;
    for (int k = 0; k < 6; ++k) out[k] = s0[k];
    F3 p = f3((float)s0[0], (float)s0[1], (float)s0[2]);
    F3 v = f3((float)s0[3], (float)s0[4], (float)s0[5]);
    float cx = (float)(s0[0] - (double)p.x), cy = (float)(s0[1] - (double)p.y),
          cz = (float)(s0[2] - (double)p.z);   // carried low part (added back)
    cx = -cx; cy = -cy; cz = -cz;               // Kahan convention: true = p - c
    const uint32_t um = P.all_mask;
    int cnt = 1, fs = -1;
    for (int i = 0; i < max_steps; ++i) {
        float valid = 3.0e38f;
        F3 dp, vn;
        if constexpr (SCHEME == 0) {                                 // integrate.hpp:55-61
            const F3 a = accel<KIND, NB>(P, um, p, v, valid);
            dp = f3(h * v.x, h * v.y, h * v.z);
            vn = f3(fmaf(h, a.x, v.x), fmaf(h, a.y, v.y), fmaf(h, a.z, v.z));
        } else {                                                     // integrate.hpp:63-93
            const float half = 0.5f * h, sixth = h / 6.f;
            F3 sx = f3(0.f, 0.f, 0.f), sv = f3(0.f, 0.f, 0.f), ps = p, vs = v;
            for (int st = 0; st < 4; ++st) {
                const F3 a = accel<KIND, NB>(P, um, ps, vs, valid);
                const float wgt = (st == 0 || st == 3) ? 1.f : 2.f;
                sx = f3(fmaf(wgt, vs.x, sx.x), fmaf(wgt, vs.y, sx.y), fmaf(wgt, vs.z, sx.z));
                sv = f3(fmaf(wgt, a.x, sv.x), fmaf(wgt, a.y, sv.y), fmaf(wgt, a.z, sv.z));
                const float c = st < 2 ? half : h;
                ps = f3(fmaf(c, vs.x, p.x), fmaf(c, vs.y, p.y), fmaf(c, vs.z, p.z));
                vs = f3(fmaf(c, a.x, v.x), fmaf(c, a.y, v.y), fmaf(c, a.z, v.z));
            }
            dp = f3(sixth * sx.x, sixth * sx.y, sixth * sx.z);
            vn = f3(fmaf(sixth, sv.x, v.x), fmaf(sixth, sv.y, v.y), fmaf(sixth, sv.z, v.z));
        }
        if (KIND == kDiffeo && !(valid > 1e-14f)) {                  // integrate.cpp:48
            fs = i;
            break;
        }
        const float yx = dp.x - cx, yy = dp.y - cy, yz = dp.z - cz;
        const F3 pn = f3(p.x + yx, p.y + yy, p.z + yz);
        cx = (pn.x - p.x) - yx;
        cy = (pn.y - p.y) - yy;
        cz = (pn.z - p.z) - yz;
        p = pn;
        v = vn;
        double* o = out + 6 * (size_t)cnt++;
        o[0] = (double)p.x - (double)cx;
        o[1] = (double)p.y - (double)cy;
        o[2] = (double)p.z - (double)cz;
        o[3] = v.x;
        o[4] = v.y;
        o[5] = v.z;
        if (use_bounds && !inside_bounds(P, p)) break;               // integrate.cpp:51
    }
    counts[r] = cnt;
    fail[r] = fs;
}

// flow_accel (integrate.hpp:46-53) at n points: acc = -Gamma(y, y), validity
// = min |det J| over the diffeo stages (1 for graph / Euclidean metrics).
template <int KIND, int NB>
__global__ void __launch_bounds__(128) accel_points_kernel(const __grid_constant__ DevParams P,
                                                           const double* __restrict__ pos,
                                                           const double* __restrict__ vel, int n,
                                                           double* __restrict__ acc,
                                                           double* __restrict__ validity) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const F3 p = f3((float)pos[3 * r], (float)pos[3 * r + 1], (float)pos[3 * r + 2]);
    const F3 v = f3((float)vel[3 * r], (float)vel[3 * r + 1], (float)vel[3 * r + 2]);
    float valid = 3.0e38f;
    const F3 a = accel<KIND, NB>(P, P.all_mask, p, v, valid);
    acc[3 * r] = a.x;
    acc[3 * r + 1] = a.y;
    acc[3 * r + 2] = a.z;
    validity[r] = KIND == kDiffeo ? (double)valid : 1.0;
}

template <int KIND, int NB>
cudaError_t trace_kind(const DevParams& P, const double* starts, int n, float h, int max_steps,
                       int scheme, int use_bounds, double* states, int* counts, int* fail,
                       cudaStream_t s) {
    const unsigned blocks = (unsigned)((n + 127) / 128);
    if (scheme == 0)
        trace_kernel<KIND, NB, 0><<<blocks, 128, 0, s>>>(P, starts, n, h, max_steps, use_bounds,
                                                          states, counts, fail);
    else
        trace_kernel<KIND, NB, 1><<<blocks, 128, 0, s>>>(P, starts, n, h, max_steps, use_bounds,
                                                          states, counts, fail);
    return cudaGetLastError();
}

} // namespace


cudaError_t launch_trace(const DevParams& P, const double* starts, int n, float h, int max_steps,
                         int scheme, int use_bounds, double* states, int* counts, int* fail,
                         cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    switch (P.kind) {
        case kEuclid:
            return trace_kind<kEuclid, 0>(P, starts, n, h, max_steps, scheme, use_bounds, states, counts, fail, s);
        case kBumps:
            return trace_kind<kBumps, 32>(P, starts, n, h, max_steps, scheme, use_bounds, states, counts, fail, s);
        case kGraphGeneral:
            return trace_kind<kGraphGeneral, 0>(P, starts, n, h, max_steps, scheme, use_bounds, states, counts, fail, s);
        default:
            return trace_kind<kDiffeo, 0>(P, starts, n, h, max_steps, scheme, use_bounds, states, counts, fail, s);
    }
}

cudaError_t launch_accel_points(const DevParams& P, const double* pos, const double* vel, int n,
                                double* acc, double* validity, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 127) / 128);
    switch (P.kind) {
        case kEuclid:
            accel_points_kernel<kEuclid, 0><<<blocks, 128, 0, s>>>(P, pos, vel, n, acc, validity);
            break;
        case kBumps:
            accel_points_kernel<kBumps, 32><<<blocks, 128, 0, s>>>(P, pos, vel, n, acc, validity);
            break;
        case kGraphGeneral:
            accel_points_kernel<kGraphGeneral, 0><<<blocks, 128, 0, s>>>(P, pos, vel, n, acc, validity);
            break;
        default:
            accel_points_kernel<kDiffeo, 0><<<blocks, 128, 0, s>>>(P, pos, vel, n, acc, validity);
    }
    return cudaGetLastError();
}

cudaError_t launch_march(const DevParams& P, const DevLaunch& L, cudaStream_t stream, int num_sms,
                         const char** kernel_name, int* launches) {
    const char* dummy;
    if (!kernel_name) kernel_name = &dummy;
    if (launches) *launches = 0;
    if (L.n_units == 0) return cudaSuccess;
    if (launches) {
        // with lights: hit + shadow launches, except the fused ray-pair kernel
        const bool lit = P.n_lights > 0 && L.mode != kModeRays;
        const bool fused = RR_RAY_PAIRS && RR_X2_FUSED &&
                           ((P.kind == kBumps && P.n_meshes == 0 &&
                             (P.scheme == 1 || (RR_RK23_PAIRS && P.scheme == 2))) ||
                            (P.scheme == 1 &&
                             RR_TWIST_PAIRS && P.kind == kDiffeo && P.n_stages == 1 &&
                             P.stages[0].kind == kStageTwist && (RR_TWIST_PAIRS_MESH || P.n_meshes == 0)) ||
                            (P.scheme == 1 && RR_CHAIN_PAIRS && P.kind == kDiffeo &&
                             !(P.n_stages == 1 && P.stages[0].kind == kStageTwist) &&
                             (RR_CHAIN_PAIRS_MESH || P.n_meshes == 0)));
        *launches = lit && !fused ? 2 : 1;
    }
    switch (P.kind) {
        case kEuclid:
            return launch_family_euclid(P, L, stream, num_sms, kernel_name);
        case kBumps:
#if RR_RAY_PAIRS
            if (P.scheme == 1 && P.n_meshes == 0)   // ray-pair frames and batches (RK4, mesh-free)
                return launch_family_pair(P, L, stream, num_sms, kernel_name);
#if RR_RK23_PAIRS
            if (P.scheme == 2 && P.n_meshes == 0)   // adaptive rk23 (EXT), mesh-free
                return launch_family_pair_rk23(P, L, stream, num_sms, kernel_name);
#endif
#endif
            return launch_family_bumps(P, L, stream, num_sms, kernel_name);
        case kGraphGeneral:
            return launch_family_graph(P, L, stream, num_sms, kernel_name);
        default:
#if RR_RAY_PAIRS && RR_TWIST_PAIRS
            // single twist, RK4: ray pairs (C4, with or without meshes)
            if (P.scheme == 1 && P.n_stages == 1 && P.stages[0].kind == kStageTwist &&
                (RR_TWIST_PAIRS_MESH || P.n_meshes == 0))
                return launch_family_pair_twist(P, L, stream, num_sms, kernel_name);
#endif
#if RR_RAY_PAIRS && RR_CHAIN_PAIRS
            // general chains, RK4: ray pairs (packed jet fold)
            if (P.scheme == 1 && !(P.n_stages == 1 && P.stages[0].kind == kStageTwist) &&
                (RR_CHAIN_PAIRS_MESH || P.n_meshes == 0))
                return launch_family_pair_chain(P, L, stream, num_sms, kernel_name);
#endif
            return launch_family_diffeo(P, L, stream, num_sms, kernel_name);
    }
}

cudaError_t launch_cull_build(const double* d_gauss, int n, int G, const double lo[3],
                              const double cell[3], double R, double dil, uint32_t* masks,
                              uint16_t* scratch, uint8_t* skip, cudaStream_t s) {
    const int cells = G * G * G;
    cull_mask_kernel<<<(cells + 255) / 256, 256, 0, s>>>(d_gauss, n, G, lo[0], lo[1], lo[2], cell[0],
                                                          cell[1], cell[2], R * R, dil, masks);
    const int lines = G * G;
    cheb_pass_kernel<<<lines, 128, G * sizeof(int), s>>>(masks, nullptr, scratch, nullptr, G, 0);
    cheb_pass_kernel<<<lines, 128, G * sizeof(int), s>>>(nullptr, scratch, scratch + cells, nullptr, G, 1);
    cheb_pass_kernel<<<lines, 128, G * sizeof(int), s>>>(nullptr, scratch + cells, nullptr, skip, G, 2);
    return cudaGetLastError();
}

cudaError_t launch_detile(const uint8_t* gathered, int width, int height, int tile_w, int tile_h,
                          int n_shards, int max_k, uint8_t* rgb, cudaStream_t stream) {
    const int tiles_x = (width + tile_w - 1) / tile_w;
    dim3 grid((width + 255) / 256, height);
    detile_kernel<<<grid, 256, 0, stream>>>(gathered, width, height, tile_w, tile_h, n_shards, max_k,
                                            tiles_x, rgb);
    return cudaGetLastError();
}

cudaError_t launch_mesh_dist(const float4* nodes, int G, const float lo[3], const float cell[3],
                             float q, uint8_t* out, cudaStream_t s) {
    const int cells = G * G * G;
    mesh_dist_kernel<<<(cells + 127) / 128, 128, 0, s>>>(nodes, G, lo[0], lo[1], lo[2], cell[0],
                                                         cell[1], cell[2], q, out);
    return cudaGetLastError();
}

bool uses_pair_kernel(const DevParams& P) {
#if RR_RAY_PAIRS
    if (P.kind == kBumps && P.n_meshes == 0) return P.scheme == 1 || (RR_RK23_PAIRS && P.scheme == 2);
    if (P.kind == kDiffeo && P.scheme == 1) {
        const bool twist1 = P.n_stages == 1 && P.stages[0].kind == kStageTwist;
        if (twist1) return RR_TWIST_PAIRS && (RR_TWIST_PAIRS_MESH || P.n_meshes == 0);
        return RR_CHAIN_PAIRS && (RR_CHAIN_PAIRS_MESH || P.n_meshes == 0);
    }
#endif
    (void)P;
    return false;
}

namespace {
__global__ void iota_kernel(unsigned* v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (unsigned)i;
}
} // namespace

size_t unit_order_temp_bytes(int n) {
    size_t b16 = 0, b32 = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, b16, (const unsigned short*)nullptr,
                                              (unsigned short*)nullptr, (const unsigned*)nullptr,
                                              (unsigned*)nullptr, n, 0, 16);
    cub::DeviceRadixSort::SortPairsDescending(nullptr, b32, (const unsigned*)nullptr, (unsigned*)nullptr,
                                              (const unsigned*)nullptr, (unsigned*)nullptr, n, 0, 16);
    return b16 > b32 ? b16 : b32;
}

cudaError_t launch_unit_order(const unsigned short* cost, unsigned short* keys_out, unsigned* iota,
                              unsigned* order, int n, void* temp, size_t temp_bytes, cudaStream_t s) {
    iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(iota, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, cost, keys_out, iota, order, n,
                                                     0, 16, s);
}

cudaError_t launch_unit_order32(const unsigned* cost, unsigned* keys_out, unsigned* iota,
                                unsigned* order, int n, void* temp, size_t temp_bytes, cudaStream_t s) {
    iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(iota, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, cost, keys_out, iota, order, n,
                                                     0, 16, s);
}

cudaError_t launch_probe(uint8_t* p, uint8_t value, cudaStream_t s) {
    probe_kernel<<<1, 1, 0, s>>>(p, value);
    return cudaGetLastError();
}

cudaError_t measure_fp32_peak(int num_sms, double* tflops) {
    float* out = nullptr;
    cudaError_t e = cudaMalloc(&out, sizeof(float));
    if (e != cudaSuccess) return e;
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    const int blocks = num_sms * 8, iters = 4096;
    ffma_peak_kernel<<<blocks, 256>>>(out, 64, 1.0000001f, 1e-7f);   // warm-up
    cudaEventRecord(t0);
    ffma_peak_kernel<<<blocks, 256>>>(out, iters, 1.0000001f, 1e-7f);
    cudaEventRecord(t1);
    e = cudaEventSynchronize(t1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * 256;
    *tflops = flops / (ms * 1e-3) / 1e12;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaFree(out);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e;
}

} // namespace rr
