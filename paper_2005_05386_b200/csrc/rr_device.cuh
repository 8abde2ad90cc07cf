// rr_device.cuh — compiled scene/metric program and the per-ray device math
// of the B200 geodesic tracer (sm_100a).
//
// Reference arithmetic this replaces (paths under /root/reference/proj):
//   raygen        src/render/camera.cpp:22-29                 -> raygen()
//   metric/Gamma  include/rray/metrics/metric.hpp:69-105,
//                 include/rray/fields/scalar_field.hpp:104-187,
//                 include/rray/fields/diffeo.hpp:111-225       -> accel_*()
//   integrator    include/rray/geodesics/integrate.hpp:46-99   -> march_unit()
//   intersection  src/render/scene.cpp:15-109                  -> intersect()
//   march loop    include/rray/render/detail/kernel_impl.hpp:22-94
//   shading       src/render/render.cpp:14-25                  -> shade()
//
// Design: one warp owns a 32-ray unit (an 8x4 pixel micro-tile
// of a frame, or 32 consecutive rays of a batch) and marches it to
// completion; warps fetch units from a global counter (persistent CTAs).
// State is register resident in FP32.  The graph metric never materialises
// Gamma: with g_j = u_j (.) s_j and v_j = a_j e_j,
//     a = (Q / (1 + |G|^2)) G,   G = sum_j v_j g_j = -grad f,
//     Q = y^T Hess(f) y = sum_j v_j [(y.g_j)^2 - sum_k y_k^2 s_jk^2],
// which is algebraically -Gamma(y,y) of metric.hpp:74-83.
// Bump parameters live in the kernel's __grid_constant__ parameter block, so
// every per-bump operand is a constant-bank operand of an FFMA.  Per step a
// warp-uniform mask (OR of the lanes' culling-cell masks) selects the bumps
// whose 7-sigma support can reach the unit's stage points.  The diffeo
// metric is evaluated as a directional jet folded innermost-first,
//     q <- D^2 Phi_s[w,w] + J_s q,  w <- J_s w,  J <- J_s J,  a = -J^-1 q,
// equal to Gamma(y,y) = J^-1 q of metric.hpp:85-100 (Theorem 1).
#pragma once

#include <cstdint>

namespace rr {

constexpr int kMaxBumps = 64;     // Gaussian terms of a graph field
constexpr int kMaxPoly = 32;      // polynomial terms of a graph field
constexpr int kMaxStages = 16;    // stages of a linearised diffeo chain
constexpr int kMaxPrims = 32;     // scene primitives
constexpr int kStaticSpheres = 4; // sphere slots evaluated with constant operands
constexpr int kStaticHalves = 2;  // half-space slots evaluated with constant operands
constexpr int kMaxLights = 8;     // point lights (EXTENSION)
constexpr int kMaxMeshes = 4;     // triangle-mesh primitives (EXTENSION)
constexpr int kUnit = 32;         // rays per warp unit
constexpr int kMicroW = 8, kMicroH = 4;   // pixel micro-tile of one warp
constexpr int kStatSlots = 11;    // 64-bit device counters per launch (DevLaunch::stats)

// g = beta * g' where g'_k = d_k * K_k, K_k = -(1/2) log2(e) / sigma_k^2.
constexpr float kBeta = -1.3862943611198906f;   // -2 ln 2
constexpr float kHalfLog2e = 0.7213475204444817f;

enum Kind : int { kEuclid = 0, kBumps = 1, kGraphGeneral = 2, kDiffeo = 3,
                  kBumpsRk23 = 4,  /* kernel-template tag only: Gaussian bumps with the adaptive
                                      rk23 scheme on the ray-pair kernel (P.kind is kBumps) */
                  kDiffeoChain = 5 /* kernel-template tag only: general diffeo chains (RK4) on
                                      the ray-pair kernel (P.kind is kDiffeo) */ };
enum Stage : int { kStageAffine = 0, kStageTwist = 1, kStageBump = 2, kStageBend = 3 };
enum Prim : int { kPrimGrid = 0, kPrimSphere = 1, kPrimHalfSpace = 2, kPrimMesh = 3 };
enum Mode : int { kModeFrame = 0, kModeTiles = 1, kModeRays = 2 };

struct DevBump {          // one Gaussian term in factored form
    float cx, cy, cz;     // centre
    float kx, ky, kz;     // K = -(1/2) log2(e) / sigma^2
    float la;             // log2 |amplitude|  (-inf for an empty slot)
    float sgn;            // sign(amplitude)
};

// One bump slot as broadcast pairs {c, c} for the ray-pair (packed FP32,
// FFMA2) march: each field is read as one 64-bit uniform operand and applies
// to both rays of a thread.  Empty slots: la = -inf, K = 0, sgn = 0.
struct alignas(8) DevBumpB {
    float2 ncx, ncy, ncz;  // -centre
    float2 kx, ky, kz;     // K
    float2 la;             // log2 |amplitude|
    float2 sgn;            // sign(amplitude)
    uint2 sgnbit;          // sign-bit mask of the amplitude (0 or 0x80000000)
    float2 kcx, kcy, kcz;  // K * centre
};

// One bump slot as scalars for the ray-pair march (RR_X2_SCALAR_CONSTS):
// the packed FP32 ops take each constant as a broadcast uniform-register
// operand (UR.F32, full rate on sm_100a: tools/microbench/fp32_pipes.cu), so
// one 64-bit uniform load brings two constants: 5 LDCU.64 per bump instead of
// DevBumpB's 10.
struct alignas(8) DevBumpS {
    float2 ncxy;           // -centre x, y
    float2 nczkx;          // -centre z, K x
    float2 kyz;            // K y, z
    float2 lakcx;          // log2 |amplitude|, (K * centre) x
    float2 kcyz;           // (K * centre) y, z
};

struct DevPoly {          // coef * x^a y^b z^c
    float coef;
    int a, b, c;
};

struct DevStage {         // one stage of a diffeo chain (identity stages dropped)
    int kind;             // kStage*
    float det;            // AFFINE: det(matrix)
    float v[12];          // AFFINE: m[9] row-major, off[3]
                          // BUMP:   cx,cy,cz, sx,sy,sz (=1/sigma), amp, dx,dy,dz
                          // BEND:   k, 1/k
    float2 v2[12];        // v as broadcast pairs {v, v} (ray-pair fold: 64-bit constant operands)
    float2 det2;
};

struct DevSphere {        // scene.cpp:56-71
    float c[3];
    float r;
    float r2;             // r*r
    float two_r;          // 2r (early-out bound)
    int index;            // position in Scene::primitives (tie-break)
    int pad;
};

struct DevHalf {          // scene.cpp:73-81: region dot(n, p) <= off
    float n[3];
    float off;
    int index;
    float inv_norm;       // 1 / |n| (free-distance bound)
    int pad[2];
};

struct DevGrid {          // scene.cpp:36-54
    float spacing, hw;
    float lo[3], hi[3];
    int index;
    int pad;
};

struct DevMesh {          // EXTENSION: BVH over a triangle soup (rr_bvh.h layouts)
    const float4* nodes;  // 2 float4 per node
    const float4* tris;   // 3 float4 per triangle
    int n_nodes, n_tris;
    int index;            // position in Scene::primitives
    int dG;               // free-distance grid: cells per axis (0: none)
    unsigned long long fingerprint;   // host: content hash (scene-change detection)
    const uint8_t* dist;  // dG^3 lower bounds of the distance from any point of a cell to the
                          // mesh (to its BVH leaf boxes), in units of dq, over the scene bounds
    float dlo[3], dinv[3];
    float dq;
    int pad2;
};

struct DevLight {
    float pos[3];
    float intensity;
};

constexpr float kShadowEps = 1e-4f;   // shadow-ray origin offset along the normal

struct alignas(16) HitRec {   // EXTENSION: primary hit for the shadow pass (32 B)
    float p[3];
    float t;
    float n[3];           // outward unit normal
    int status;           // 0 miss, 1 hit, 2 failed
};

struct DevParams {
    int kind;             // Kind
    int n_bumps, n_poly, n_stages;
    int n_prims, n_lights, scheme, max_steps;
    int n_spheres, n_halves, n_grids, n_meshes;
    int nb_slot;          // kBumps: bump slots of the kernel variant (4/8/16/32)
    float h, fog;
    float inv_h;          // 1 / h
    float ambient;        // EXTENSION: lit shading ambient term
    float tol;            // EXTENSION: rk23 error tolerance
    float lo[3], hi[3];   // scene bounds
    int cull;             // 1: cull_masks valid
    int grid;             // culling voxels per axis
    float grid_lo[3], grid_inv[3];
    uint32_t all_mask;    // bits of every live bump (slot bits for kBumps)
    uint32_t neg_mask;    // slots with a negative amplitude (kBumps)
    const uint32_t* cull_masks;   // grid^3 bump masks (device); rk23: 3 levels
    unsigned cull_cells;          // grid^3 (level stride)
    const uint8_t* skip_k;        // grid^3 Chebyshev distance (cells) to the nearest non-empty cell
    int skip;                     // 1: empty-space skipping enabled
    float cell_min;               // smallest culling-cell edge (world units)
    DevBump bumps[kMaxBumps];
    DevBumpB bumpsb[32];              // slots 0..31 as broadcast pairs (ray-pair march)
    DevBumpS bumpss[32];              // slots 0..31 as scalar pairs (ray-pair march, UR.F32 operands)
    DevPoly poly[kMaxPoly];
    DevStage stages[kMaxStages];
    DevSphere spheres[kMaxPrims];
    DevHalf halves[kMaxPrims];
    DevGrid grids[kMaxPrims];
    DevMesh meshes[kMaxMeshes];
    DevLight lights[kMaxLights];
};

struct DevCamera {        // render::Camera in device form (camera.hpp:15-30)
    double pos[3];
    double f0[3], f1[3], f2[3];   // look, up, right (g-orthonormal)
    double g[6];                  // xx,xy,xz,yy,yz,zz at pos
    double tan_half, aspect;
};

struct DevLaunch {
    DevCamera cam;
    int mode;                     // Mode
    int width, height;
    int tile_w, tile_h;           // tile mode: tile size (multiples of 8x4)
    int shard, n_shards;
    int tiles_x;                  // tiles per frame row
    int micro_per_tile;           // (tile_w/8)*(tile_h/4)
    unsigned n_units;             // warp units of this launch
    int lpp;                      // shadow pass: lights marched per pixel in one unit (1/2/4)
    uint8_t* rgb;                 // frame (row-major) or tile-major buffer
    const double* rays;           // RAYS: 6 doubles per ray (RayStart)
    uint8_t* outcomes;            // 48-byte PixelOutcome records: RAYS (by ray), frames when
                                  // non-null (outcome sink, row-major pixel index)
    int vec16;                    // ray-pair epilogue may store 16x4 RGB blocks as 16-B words
    int vec8;                     // one-ray epilogue may store 8x4 RGB micro-tiles as 8-B words
    const unsigned* order;        // ray-pair kernels: dispatch order of the primary units
                                  // (expensive first, from the previous frame's costs) or null
    unsigned short* unit_cost;    // ray-pair kernels: warp-loop iterations per primary unit (or null)
    const unsigned* order2;       // fused lit launch: dispatch order of the units' shadow items
    unsigned* unit_cost2;         // fused lit launch: shadow iterations per unit (max over lights;
                                  // zeroed per launch)
    unsigned long long out_pixels;    // pixels of the rgb / hit-record buffers (RR_CHECKS bounds)
    unsigned long long n_outcomes;    // records of the outcome sink (RR_CHECKS bounds)
    unsigned long long n_rays;
    unsigned* counter;            // unit dispensers [2] (zeroed per launch)
    unsigned long long* stats;    // [0] steps [1] errors [2] integrated [3] bump evals [4] rays
                                  // [5] shadow steps [6] lane slots [7] shadow lane slots
                                  // [8] jumps [9] shadow jumps [10] shadow integrated
                                  // (kStatSlots entries)
    HitRec* hits;                 // EXTENSION: hit records (lights present)
    unsigned* done;               // EXTENSION: lights finished per ray-pair unit (zeroed per launch)
    uint8_t* vis;                 // EXTENSION: light visibility per (pixel, light)
    unsigned* ready;              // EXTENSION: fused launch: hit records of a pair unit written
};

} // namespace rr
