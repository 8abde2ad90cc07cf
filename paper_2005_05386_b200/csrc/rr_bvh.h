// rr_bvh.h — host-side BVH build for triangle-mesh primitives (EXTENSION;
// "Host SAH build; top levels staged on the device").
#pragma once

#include <cstdint>
#include <vector>

namespace rr {

// Device records produced by build_bvh (see rr_device.cuh DevMesh):
//   node (8 floats, 32 B): lo.xyz, a | hi.xyz, b   (a, b are int bit patterns)
//       leaf:  b > 0, triangles [a, a + b) of the triangle array
//       inner: b == 0, left child = this + 1, right child = a
//   triangle (12 floats, 48 B): v0.xyz, original index | e1.xyz, 0 | e2.xyz, 0
struct BvhBuild {
    std::vector<float> nodes;   // 8 per node, depth-first (left child follows its parent)
    std::vector<float> tris;    // 12 per triangle, in leaf order
    int depth = 0;
};

// Binned SAH (12 bins on each axis, leaves of <= 4 triangles).
void build_bvh(const double* vertices, int n_vertices, const int32_t* triangles, int n_triangles,
               BvhBuild& out);

} // namespace rr
