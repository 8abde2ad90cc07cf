// rr_internal.h — host-side interface between the C-ABI layer (rr_host.cpp)
// and the kernel launchers (rr_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "rr_device.cuh"

namespace rr {

// Launches the fused raygen+march+shade kernel variant matching P (kind,
// bump capacity, scheme).  L.counter / L.stats must already be zeroed on
// `stream`.  Returns cudaSuccess or the launch error.
cudaError_t launch_march(const DevParams& P, const DevLaunch& L, cudaStream_t stream,
                         int num_sms, const char** kernel_name, int* launches = nullptr);

// Per-family march launchers (one translation unit each, see rr_march.cuh);
// launch_march dispatches on P.kind.
cudaError_t launch_family_pair(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                               const char** name);
cudaError_t launch_family_pair_twist(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                     const char** name);
cudaError_t launch_family_pair_rk23(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                    const char** name);
cudaError_t launch_family_pair_chain(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                     const char** name);
cudaError_t launch_family_bumps(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                const char** name);
cudaError_t launch_family_diffeo(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                 const char** name);
cudaError_t launch_family_euclid(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                 const char** name);
cudaError_t launch_family_graph(const DevParams& P, const DevLaunch& L, cudaStream_t s, int sms,
                                const char** name);

// Builds the culling grid (bump masks + Chebyshev distances) on the device:
// d_gauss holds n records {cx, cy, cz, sigma_x, sigma_y, sigma_z, slot, pad}.
// scratch needs 2*G^3 uint16.  4 launches on `s`.
cudaError_t launch_cull_build(const double* d_gauss, int n, int G, const double lo[3],
                              const double cell[3], double R, double dil, uint32_t* masks,
                              uint16_t* scratch, uint8_t* skip, cudaStream_t s);

// Reassembles a row-major frame from gathered tile-major shard buffers.
cudaError_t launch_detile(const uint8_t* gathered, int width, int height, int tile_w,
                          int tile_h, int n_shards, int max_tiles_per_shard, uint8_t* rgb,
                          cudaStream_t stream);

// Off the render path: trace_geodesic polylines (scheme 0 Euler / 1 RK4;
// states n x (max_steps+1) x 6 doubles) and flow_accel at n points, all
// device buffers, on `s`.
cudaError_t launch_trace(const DevParams& P, const double* starts, int n, float h, int max_steps,
                         int scheme, int use_bounds, double* states, int* counts, int* fail,
                         cudaStream_t s);
cudaError_t launch_accel_points(const DevParams& P, const double* pos, const double* vel, int n,
                                double* acc, double* validity, cudaStream_t s);

// True when launch_march runs a ray-pair (march2) kernel for P.
bool uses_pair_kernel(const DevParams& P);

// Expensive-first dispatch order of ray-pair units: order = unit ids sorted
// by descending cost (device radix sort on 16-bit keys, on `s`).
size_t unit_order_temp_bytes(int n);
cudaError_t launch_unit_order(const unsigned short* cost, unsigned short* keys_out, unsigned* iota,
                              unsigned* order, int n, void* temp, size_t temp_bytes, cudaStream_t s);

cudaError_t launch_unit_order32(const unsigned* cost, unsigned* keys_out, unsigned* iota,
                                unsigned* order, int n, void* temp, size_t temp_bytes, cudaStream_t s);

// Mesh free-distance grid (G^3 bytes, units of q) over the box lo + [0, G cell).
cudaError_t launch_mesh_dist(const float4* nodes, int G, const float lo[3], const float cell[3],
                             float q, uint8_t* out, cudaStream_t s);

// One-byte device store (+ system fence) through a possibly peer/IPC-mapped
// pointer: the exchange's mapping probe.
cudaError_t launch_probe(uint8_t* p, uint8_t value, cudaStream_t s);

// Dense FFMA microbenchmark; returns TFLOP/s (2 flop per FFMA).
cudaError_t measure_fp32_peak(int num_sms, double* tflops);

// Number of micro-tiles (warp units) covering tile k of a tiling.
inline int micro_per_tile(int tile_w, int tile_h) {
    return (tile_w / kMicroW) * (tile_h / kMicroH);
}

} // namespace rr
