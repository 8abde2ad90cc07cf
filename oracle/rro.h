/*
 * rro.h — FP64 CPU ORACLE (test infrastructure only; never the product).
 *
 * A plain-C restatement of the reference's per-pixel geodesic tracing path
 * (/root/reference/proj), operating on the same flattened descriptors as the
 * product C-ABI (include/rray_cuda.h).  Each function cites the reference
 * file:line it restates and keeps the reference's operation order, so with
 * -ffp-contract=off it reproduces the reference bit for bit; that identity
 * is pinned by tests/test_oracle.py against golden vectors dumped from the
 * reference itself (tests/golden/make_golden.py via oracle/_ref).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.
 */
#ifndef RRO_H
#define RRO_H

#include <stddef.h>
#include <stdint.h>

#include "rray_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Flags produced by rro_flags (parity harness). */
enum {
    RRO_FLAG_GRAZING = 1,   /* status/prim changes under +-perturbation of the direction */
    RRO_FLAG_WRAP = 2,      /* some hit coordinate lies within wrap_eps of an integer */
    RRO_FLAG_LIMIT = 4,     /* outcome flips if the march were one step longer / shorter */
    RRO_FLAG_WRAP_X = 8,    /* per-channel wrap bits: R, G, B individually */
    RRO_FLAG_WRAP_Y = 16,
    RRO_FLAG_WRAP_Z = 32,
    RRO_FLAG_SHADOW = 64    /* EXT: a light's visibility flips under shadow-ray perturbation */
};

const char* rro_last_error(void);

/* integrate.hpp:46-53 */
void rro_flow_accel(const rr_metric_desc* m, const double pos[3], const double vel[3],
                    double acc[3], double* validity);
/* integrate.hpp:55-99; state = pos[3], vel[3] */
void rro_step(const rr_metric_desc* m, const double s[6], double h, int scheme, double out[6],
              double* validity);
/* scene.cpp:99-109; returns 1 on hit */
int rro_intersect(const rr_scene_desc* sc, const double a[3], const double b[3],
                  double point[3], double* s, int* prim);
/* kernel_impl.hpp:22-94 (scalar lane type) over n rays, OpenMP `threads` */
void rro_march(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_integrator* integ,
               const rr_ray_start* rays, rr_pixel_outcome* out, size_t n, int threads);
/* camera.cpp:9-20; 0 ok, 2 numeric (DegenerateBasis / singular metric) */
int rro_build_camera(const rr_metric_desc* m, const double pos[3], const double look[3],
                     const double up[3], double fov, rr_camera* out);
/* camera.cpp:22-29 */
void rro_pixel_direction(const rr_camera* cam, int px, int py, int w, int h, double out[3]);
/* render.cpp:14-25 (+ magenta for failures, render.cpp:39,81-83) */
void rro_shade_outcome(const rr_pixel_outcome* o, double kappa, uint8_t rgb[3]);
/* render.cpp:43-111: rgb (3*w*h) and optional per-pixel outcomes */
void rro_render(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_camera* cam,
                const rr_integrator* integ, int w, int h, uint8_t* rgb,
                rr_pixel_outcome* outcomes, rr_stats* stats, int threads);
/* Parity flags per pixel for a rendered frame. */
void rro_flags(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_camera* cam,
               const rr_integrator* integ, int w, int h, const rr_pixel_outcome* outcomes,
               double perturb_rad, double wrap_eps, uint8_t* flags, int threads);

/* Rows row0, row0 + row_step, ... of the w x h frame (output row k = frame
 * row row0 + k row_step); rgb_rows / outcome_rows may be NULL. */
void rro_render_rows(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_camera* cam,
                     const rr_integrator* integ, int w, int h, int row0, int row_step,
                     uint8_t* rgb_rows, rr_pixel_outcome* outcome_rows, rr_stats* stats,
                     int threads);
/* Parity flags of a list of pixels (row-major indices pix[k], FP64 outcome
 * outcomes[k]); same flags as rro_flags. */
void rro_flags_pixels(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_camera* cam,
                      const rr_integrator* integ, int w, int h, const int64_t* pix,
                      const rr_pixel_outcome* outcomes, size_t n, double perturb_rad,
                      double wrap_eps, uint8_t* flags, int threads);

/* Test hook: 1 = mesh intersection scans every triangle (no BVH pruning). */
void rro_set_mesh_bruteforce(int on);

#ifdef __cplusplus
}
#endif
#endif
