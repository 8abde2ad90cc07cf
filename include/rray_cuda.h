/*
 * rray_cuda.h — C-ABI of the B200-native geodesic ray tracer.
 *
 * This is the drop-in boundary for the reference's per-pixel geodesic
 * tracing path (arxiv/paper_2005_05386, the `rray` C++20 CPU renderer under
 * /root/reference/proj).  Every entry point below replaces one reference
 * interface; the comment on each cites the reference file:line it stands in
 * for.  INTEGRATION.md shows the reference-side binding a maintainer adds
 * (a `KernelKind::Cuda` MarchFn thunk plus a whole-frame `render()` route).
 *
 * Conventions
 *  - Plain C: no C++ or torch types cross this boundary; pointers + sizes.
 *  - Every function returns an int status with the reference CLI's exit-code
 *    meaning (tools/rray_main.cpp:185-194):
 *        0 ok, 1 config/validation, 2 numeric, 3 I/O,
 *    plus one extension, 4 = device/runtime (CUDA) failure.  The message of
 *    the last failure on a context is available from rr_last_error().
 *  - Host-side records are byte-compatible with the reference structs so a
 *    MarchFn shim can pass its buffers straight through:
 *        rr_ray_start     == render::RayStart      (kernel.hpp:26-29, 48 B)
 *        rr_pixel_outcome == render::PixelOutcome  (kernel.hpp:33-39, 48 B)
 *        rr_vec3          == core::Vec3            (linalg.hpp:18-26, 24 B)
 *  - Scene and metric expression trees (std::variant trees in the reference,
 *    scalar_field.hpp:49-64, diffeo.hpp:57-104, metric.hpp:34-49,
 *    scene.hpp:43-51) are passed flattened into node arrays; children are
 *    referenced through one shared index array.
 *
 * Thread safety: a context may be used from many host threads at once (the
 * reference calls MarchFn concurrently from RRAY_THREADS workers,
 * render.cpp:29-37, :67-104); calls on one context are serialised
 * internally, and every call sets the context's device first, whatever the
 * calling thread's current device.  Asynchronous *_device calls on one
 * context may use different streams: a launch on a new stream waits for the
 * context's previous launch (they share the dispatch counter and scratch).
 */
#ifndef RRAY_CUDA_H
#define RRAY_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RR_ABI_VERSION 1

/* ---- status codes (rray_main.cpp:185-194) ------------------------------- */
enum {
    RR_OK = 0,
    RR_ERR_CONFIG = 1,  /* ConfigError / ValidationError (error.hpp:29-44) */
    RR_ERR_NUMERIC = 2, /* NumericError family (error.hpp:13-27) */
    RR_ERR_IO = 3,      /* IoError (error.hpp:47-50) */
    RR_ERR_DEVICE = 4   /* extension: CUDA runtime / device failure */
};

/* ---- geometry ------------------------------------------------------------ */
typedef struct rr_vec3 { double x, y, z; } rr_vec3;          /* core::Vec3 */
typedef struct rr_aabb { rr_vec3 min, max; } rr_aabb;        /* core::Aabb (aabb.hpp:7-22) */

/* ---- scalar fields f: R^3 -> R (scalar_field.hpp:16-64) ------------------ */
typedef struct rr_gaussian {          /* fields::GaussianParams :16-22 */
    double amplitude;
    rr_vec3 center;
    rr_vec3 sigma;                    /* all > 0 */
} rr_gaussian;

typedef struct rr_poly_term {         /* fields::PolyTerm :25-30 */
    double coef;
    int32_t powers[3];                /* total degree <= 4 (config.cpp:181) */
    int32_t pad_;
} rr_poly_term;

enum { RR_FIELD_GAUSSIAN = 0, RR_FIELD_POLYNOMIAL = 1, RR_FIELD_SUM = 2 };

typedef struct rr_field_node {        /* one ScalarFieldExpr node */
    int32_t kind;                     /* RR_FIELD_* */
    int32_t first;                    /* POLYNOMIAL: first poly_terms index; SUM: first children index */
    int32_t count;                    /* POLYNOMIAL: #terms; SUM: #children (field node indices) */
    int32_t pad_;
    rr_gaussian gaussian;             /* GAUSSIAN only */
} rr_field_node;

/* ---- diffeomorphisms Phi: R^3 -> R^3 (diffeo.hpp:59-104) ----------------- */
enum {
    RR_DIFFEO_IDENTITY = 0,
    RR_DIFFEO_AFFINE = 1,
    RR_DIFFEO_TWIST = 2,
    RR_DIFFEO_LOCAL_BUMP = 3,
    RR_DIFFEO_COMPOSE = 4,
    RR_DIFFEO_BEND = 5      /* EXTENSION: Barr bend about z, angle = curvature * x (see rro.c) */
};

typedef struct rr_diffeo_node {       /* one DiffeoExpr node */
    int32_t kind;                     /* RR_DIFFEO_* */
    int32_t first;                    /* COMPOSE: first children index; maps[0] is the OUTERMOST map */
    int32_t count;                    /* COMPOSE: #maps (>= 1) */
    int32_t pad_;
    double matrix[3][3];              /* AFFINE: row-major (linalg.hpp:172-174) */
    rr_vec3 offset;                   /* AFFINE */
    rr_gaussian bump;                 /* LOCAL_BUMP: Phi(p) = p + f(p) * direction */
    rr_vec3 direction;                /* LOCAL_BUMP */
    double curvature;                 /* BEND (EXTENSION) */
} rr_diffeo_node;

/* ---- metric fields (metric.hpp:20-49) ------------------------------------ */
enum { RR_METRIC_EUCLIDEAN = 0, RR_METRIC_GRAPH = 1, RR_METRIC_DIFFEO = 2 };

typedef struct rr_metric_desc {
    int32_t kind;                     /* RR_METRIC_* */
    int32_t root;                     /* GRAPH: root field node; DIFFEO: root diffeo node */
    int32_t n_field_nodes;
    int32_t n_poly_terms;
    int32_t n_diffeo_nodes;
    int32_t n_children;
    const rr_field_node* field_nodes;
    const rr_poly_term* poly_terms;
    const rr_diffeo_node* diffeo_nodes;
    const int32_t* children;
} rr_metric_desc;

/* ---- scene (scene.hpp:18-51) --------------------------------------------- */
enum { RR_PRIM_GRID_PLANES = 0, RR_PRIM_SPHERE = 1, RR_PRIM_HALF_SPACE = 2,
       RR_PRIM_MESH = 3 /* EXTENSION: triangle mesh (SPEC.md:491 lists it as a non-goal) */ };

typedef struct rr_primitive {
    int32_t kind;                     /* RR_PRIM_* */
    int32_t pad_;
    double spacing, half_width;       /* GRID_PLANES (scene.hpp:20-26) */
    rr_aabb bounds;                   /* GRID_PLANES clip box */
    rr_vec3 center;                   /* SPHERE (scene.hpp:28-33) */
    double radius;
    rr_vec3 normal;                   /* HALF_SPACE: region dot(normal,p) <= offset (scene.hpp:35-41) */
    double offset;
    /* MESH (EXTENSION): a triangle soup, hit like the other primitives by
     * the chord [a, b] of each step (nearest s in [0, 1]; ties between
     * triangles keep the lower triangle index); no inside-start rule (a
     * surface, not a solid).  The library builds and owns its BVH. */
    int32_t n_vertices, n_triangles;
    const double* vertices;           /* n_vertices * 3 */
    const int32_t* triangles;         /* n_triangles * 3 vertex indices */
} rr_primitive;

/* Point light (EXTENSION: shadow geodesics; no reference counterpart,
 * SPEC.md:491,494).  n_lights == 0 selects the reference shading exactly.
 * With lights, a hit at q with outward unit normal n is shaded
 *     I = ambient + sum_l intensity_l * lambert_l * lit_l,
 *     lambert_l = n . (L_l - q) / |L_l - q|   (no shadow ray when <= 0),
 *     channel = lround(255 * frac(x) * exp(-kappa t) * I)  clamped to [0,255],
 * where lit_l comes from a shadow geodesic started at q + 1e-4 n with unit
 * g-speed along L_l - q, marched with the frame's integrator: blocked when a
 * primitive is hit closer to q than |L_l - q|, lit when it crosses that
 * sphere, leaves the bounds or exhausts max_steps (oracle/rro.c
 * shadow_march is the FP64 definition). */
typedef struct rr_light {
    rr_vec3 position;
    double intensity;
} rr_light;

typedef struct rr_scene_desc {
    int32_t n_primitives;
    int32_t n_lights;                 /* EXTENSION; 0 for reference scenes */
    const rr_primitive* primitives;
    const rr_light* lights;
    rr_aabb bounds;                   /* rays terminate once they leave it */
    double fog_density;               /* kappa of exp(-kappa t) (render.cpp:14-25) */
    double ambient;                   /* EXTENSION: ambient term of the lit shading (n_lights > 0) */
} rr_scene_desc;

/* ---- integrator (integrate.hpp:30-36) ------------------------------------ */
enum { RR_SCHEME_EULER = 0, RR_SCHEME_RK4 = 1,
       RR_SCHEME_RK23 = 2 /* EXTENSION: adaptive Bogacki-Shampine 3(2), see oracle/rro.c */ };

typedef struct rr_integrator {
    double h;                         /* step (RK23: initial step; steps stay in [h/64, 4h]) */
    int32_t max_steps;                /* RK23: accepted steps */
    int32_t scheme;                   /* RR_SCHEME_* */
    double tol;                       /* RK23 (EXTENSION): abs+rel error tolerance per step */
} rr_integrator;

/* ---- march records (kernel.hpp:26-45) ------------------------------------ */
enum { RR_MISS = 0, RR_HIT = 1, RR_FAILED = 2 };   /* render::RayStatus */

typedef struct rr_ray_start {         /* render::RayStart, 48 B */
    rr_vec3 position;
    rr_vec3 direction;                /* unit g-speed */
} rr_ray_start;

typedef struct rr_pixel_outcome {     /* render::PixelOutcome, 48 B */
    uint8_t status;                   /* RR_MISS / RR_HIT / RR_FAILED */
    int32_t prim;                     /* hit primitive index, -1 otherwise */
    rr_vec3 point;                    /* hit point */
    double t;                         /* (step + s) * h */
    int32_t steps;
} rr_pixel_outcome;

/* ---- camera (camera.hpp:15-30) ------------------------------------------- */
typedef struct rr_camera {            /* render::Camera, same field order */
    rr_vec3 position;
    rr_vec3 look_dir;
    rr_vec3 up_hint;
    double fov;                       /* vertical, radians */
    rr_vec3 frame[3];                 /* g-orthonormal: look, up, right */
    double g[6];                      /* g at position, SymMat3 xx,xy,xz,yy,yz,zz */
} rr_camera;

/* ---- statistics (render.hpp:24-33) ---------------------------------------- */
typedef struct rr_stats {
    double wall_seconds;
    int64_t rays;
    int64_t total_steps;              /* reference semantics: sum of PixelOutcome.steps */
    int64_t pixel_errors;             /* magenta pixels */
    /* extensions (device-side accounting) */
    double device_ms;                 /* CUDA-event time of the march launch(es) */
    int64_t integrated_steps;         /* steps the device actually integrated (a straight jump
                                         through metric-free space counts once), all passes */
    int64_t bump_evals;               /* Gaussian-term evaluations executed (N_eff accounting) */
    int64_t shadow_steps;             /* steps spent on shadow geodesics (EXT) */
    int64_t kernel_launches;          /* kernels the call launched (march + the dispatch-order sort) */
    int64_t lane_slots;               /* primary: warp loop iterations x 32 (SIMT efficiency = integrated / slots) */
    int64_t shadow_lane_slots;        /* same for the shadow pass (EXT) */
    int64_t jump_steps;               /* primary integrated steps that were straight jumps through
                                         metric-free space (no RK4 / metric evaluation) */
    int64_t shadow_jump_steps;        /* same for the shadow pass (EXT) */
    int64_t shadow_integrated_steps;  /* the shadow pass's share of integrated_steps (EXT) */
    int64_t sort_kernels;             /* of kernel_launches: the dispatch-order sort's kernels
                                         (rr_options.order_units); the rest are march launches */
} rr_stats;

/* ---- tuning knobs (extension; defaults are parity-safe) ------------------- */
typedef struct rr_options {
    int32_t cull;                     /* per-warp bump culling on a voxel grid: 0 off, 1 (default)
                                         radius cull_radius_sigma for every bump, 2 equal-error
                                         radii <= cull_radius_sigma (see ensure_masks) */
    int32_t cull_grid;                /* voxels per axis of the culling grid (default 256) */
    double cull_radius_sigma;         /* bump support radius in sigmas (default 5.5) */
    int32_t block_x, block_y;         /* frame tile ordering the warp units (default 32 x 32) */
    int32_t persistent;               /* 1: persistent CTAs pulling warp units (default 1) */
    int32_t skip;                     /* 1: empty-space skipping of bump-free cells (default 1) */
    int32_t order_units;              /* 1: ray-pair frames dispatch their units expensive-first,
                                         ordered by the previous launch's per-unit cost with the
                                         same unit layout (default 1; outputs are unaffected) */
} rr_options;

typedef struct rr_ctx rr_ctx;

/* Library/ABI identification. */
int rr_abi_version(void);
const char* rr_build_info(void);

/* Context lifetime.  `device` is a CUDA ordinal (one process per GPU).
 * Replaces the implicit global state of march_fn() (kernel_dispatch.cpp:40-54). */
int rr_create(rr_ctx** out, int device);
void rr_destroy(rr_ctx* ctx);
const char* rr_last_error(const rr_ctx* ctx);
int rr_set_options(rr_ctx* ctx, const rr_options* opt);
int rr_get_options(const rr_ctx* ctx, rr_options* opt);

/* Uploads a flattened metric + scene.  Replaces the borrowed variant trees of
 * MarchContext (kernel.hpp:41-45); validates them like config.cpp:144-338. */
int rr_set_scene(rr_ctx* ctx, const rr_metric_desc* metric, const rr_scene_desc* scene);

/* render::build_camera (camera.cpp:9-20) against the context's metric.
 * fov in radians.  Status 2 on DegenerateBasis / singular metric. */
int rr_build_camera(rr_ctx* ctx, const rr_vec3* position, const rr_vec3* look_dir,
                    const rr_vec3* up_hint, double fov, rr_camera* out);

/* render::pixel_direction (camera.cpp:22-29); host helper for MarchFn callers. */
int rr_pixel_direction(const rr_camera* cam, int px, int py, int width, int height,
                       rr_vec3* out);

/* MarchFn-compatible batch (kernel.hpp:47, march_rays kernel_impl.hpp:96-108):
 * host buffers, out[0..n) fully written.  Safe to call concurrently. */
int rr_march(rr_ctx* ctx, const rr_integrator* integ, const rr_ray_start* rays,
             rr_pixel_outcome* out, size_t n);

/* Same with device-resident buffers on a caller stream (cudaStream_t or NULL). */
int rr_march_device(rr_ctx* ctx, const rr_integrator* integ, const rr_ray_start* d_rays,
                    rr_pixel_outcome* d_out, size_t n, void* stream);

/* Whole-frame render (render::render, render.cpp:43-111): device raygen +
 * march + shade, RGB8 row-major into a HOST buffer of 3*w*h bytes.  When the
 * buffer is page-locked (cudaHostAlloc / cudaHostRegister / torch
 * pin_memory) the kernel writes the pixels straight into it through its UVA
 * mapping; pageable buffers get a device->host copy after the kernel. */
int rr_render(rr_ctx* ctx, const rr_camera* cam, const rr_integrator* integ, int width,
              int height, uint8_t* rgb_out, rr_stats* stats);

/* Whole frame with per-pixel outcomes (parity entry of the frame path): the
 * SAME frame kernel rr_render launches (device raygen, march, shade) also
 * writes each pixel's render::PixelOutcome record (kernel.hpp:33-39, the
 * records render.cpp:68-84 shades), row-major, into `out` (w*h records).
 * `rgb_out` (3*w*h bytes) may be NULL.  With lights the outcome is the
 * primary ray's (the shadow pass only shades). */
int rr_render_outcomes(rr_ctx* ctx, const rr_camera* cam, const rr_integrator* integ, int width,
                       int height, uint8_t* rgb_out, rr_pixel_outcome* out, rr_stats* stats);

/* Whole-frame render into a DEVICE buffer on a caller stream.  When `stats`
 * is non-NULL the call synchronises the stream to fill it; pass NULL for
 * asynchronous back-to-back frames. */
int rr_render_device(rr_ctx* ctx, const rr_camera* cam, const rr_integrator* integ,
                     int width, int height, uint8_t* d_rgb, rr_stats* stats, void* stream);

/* Multi-GPU tile sharding.  The frame is cut into tile_w x
 * tile_h tiles numbered row-major; shard `shard` of `n_shards` renders tiles
 * i with i % n_shards == shard into d_tiles, tile-major (tile k of this
 * shard at byte offset k * 3*tile_w*tile_h, pixels row-major inside the
 * tile; partial edge tiles are padded with zeros). */
int rr_shard_tile_count(int width, int height, int tile_w, int tile_h, int shard,
                        int n_shards);
int rr_render_tiles(rr_ctx* ctx, const rr_camera* cam, const rr_integrator* integ, int width,
                    int height, int tile_w, int tile_h, int shard, int n_shards,
                    uint8_t* d_tiles, rr_stats* stats, void* stream);

/* Fused render + exchange: renders shard `shard`'s tiles (same tiling as
 * rr_render_tiles) and writes each pixel straight to its place in a
 * row-major RGB8 frame d_frame, which may live on ANOTHER GPU (a CUDA-IPC /
 * peer mapping of rank 0's frame: the shade epilogue's stores travel over
 * NVLink, no gather or detile pass).  Visibility to the frame's owner
 * follows kernel completion plus a cross-rank synchronisation.  As for every
 * `stream` argument, NULL selects the context's own NON-BLOCKING stream,
 * which is not ordered after work on the legacy default stream: initialise
 * d_frame (if at all) and synchronise before the call. */
int rr_render_shard(rr_ctx* ctx, const rr_camera* cam, const rr_integrator* integ, int width,
                    int height, int tile_w, int tile_h, int shard, int n_shards,
                    uint8_t* d_frame, rr_stats* stats, void* stream);

/* ---- cross-process / cross-device frame exchange ----------
 * The reference renders in one process (render.cpp:96-104); on a multi-GPU
 * node one process drives each GPU and rr_render_shard's epilogue stores its
 * pixels straight into rank 0's frame.  These calls make that mapping the
 * library's business: the frame's owner exports its device buffer, every
 * other process imports it ON ITS OWN CONTEXT'S DEVICE (cudaIpcOpenMemHandle
 * with lazy peer access, after enabling peer access where the devices
 * support it), proves the mapping with a device-side store, and closes it
 * before the owner frees the frame. */
typedef struct rr_frame_handle {
    unsigned char ipc[64];            /* cudaIpcMemHandle_t of the allocation holding the frame */
    uint64_t offset;                  /* byte offset of the frame inside that allocation */
    uint64_t bytes;                   /* frame size in bytes */
    uint64_t ptr;                     /* exporter's device address (same-process imports) */
    int32_t device;                   /* exporter's CUDA ordinal */
    int32_t pid;                      /* exporter's process id */
} rr_frame_handle;

/* Handle for `bytes` of device memory at d_frame (on ctx's device; any
 * cudaMalloc'd or caching-allocator sub-allocation). */
int rr_frame_export(rr_ctx* ctx, const void* d_frame, size_t bytes, rr_frame_handle* out);
/* Maps an exported frame into this context's device; *d_frame is a device
 * address usable as rr_render_shard's d_frame on ctx's device. */
int rr_frame_import(rr_ctx* ctx, const rr_frame_handle* h, void** d_frame);
/* Unmaps an imported frame (no-op for same-process imports). */
int rr_frame_close(rr_ctx* ctx, void* d_frame);
/* One device-side store of `value` at d_frame + offset from ctx's device,
 * fenced system-wide and synchronised: a failing mapping returns status 4
 * instead of faulting the first frame. */
int rr_frame_probe(rr_ctx* ctx, void* d_frame, size_t offset, uint8_t value);

/* Reassembles a frame from the concatenation of every shard's tile buffer
 * (shard 0 first, each padded to the largest shard's tile count). */
int rr_detile(rr_ctx* ctx, const uint8_t* d_gathered, int width, int height, int tile_w,
              int tile_h, int n_shards, uint8_t* d_rgb, void* stream);

/* ---- Off the render path: geodesic export and device verify ------------
 * (`python -m paper_2005_05386_b200 geodesic|verify`). */

/* trace_geodesic (src/geodesics/integrate.cpp:40-54) on the device, one
 * geodesic per start, scheme euler|rk4 with step integ->h for up to
 * integ->max_steps steps.  states: n x (max_steps+1) x 6 doubles
 * {x, y, z, vx, vy, vz} (state i at t = i h; states[0] = the start);
 * counts[r] = states written (the exiting state is kept when use_bounds and
 * the scene bounds are left, integrate.cpp:51); fail_step[r] = the step whose
 * metric evaluation failed (|det J| <= 1e-14, integrate.cpp:48: the
 * reference throws NumericError naming it) or -1. */
int rr_trace(rr_ctx* ctx, const rr_integrator* integ, const rr_ray_start* starts, size_t n,
             int use_bounds, double* states, int32_t* counts, int32_t* fail_step);

/* flow_accel (include/rray/geodesics/integrate.hpp:46-53) evaluated by the
 * device metric program at n points: acc = -Gamma(vel, vel) (n x 3) and the
 * validity (min |det J|; 1 for graph / Euclidean metrics). */
int rr_accel(rr_ctx* ctx, const double* pos, const double* vel, size_t n, double* acc,
             double* validity);

/* FP64 host metric tensor g(p) as {xx, xy, xz, yy, yz, zz}
 * (src/metrics/metric.cpp:12-15, :40-42); status 2 when singular. */
int rr_metric_tensor(rr_ctx* ctx, const double* p, double* g);

/* FP64 finite-difference Christoffel oracle (src/metrics/metric.cpp:88-133,
 * step h_fd, reference default 1e-4): gamma[6 m + q] = Gamma^m in the
 * SymMat3 order {xx, xy, xz, yy, yz, zz}. */
int rr_christoffel_fd(rr_ctx* ctx, const double* p, double h_fd, double* gamma);

/* FP64 image Phi(p) of the diffeo chain (eval_diffeo_raw, diffeo.hpp:214-225;
 * p itself for graph / Euclidean metrics). */
int rr_diffeo_image(rr_ctx* ctx, const double* p, double* image);

/* Microbenchmark of the FP32 FMA pipe (roofline denominator): returns the
 * measured dense FFMA throughput of this device in TFLOP/s. */
int rr_measure_fp32_peak(rr_ctx* ctx, double* tflops);

/* Diagnostics: name of the kernel variant the context's last launch used
 * (e.g. "march2_kernel<bumps16>"); "" before the first launch.  The
 * reference has no counterpart (its KernelKind is chosen, not reported). */
const char* rr_last_kernel(const rr_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* RRAY_CUDA_H */
