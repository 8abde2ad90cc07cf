/*
 * rro.c — FP64 CPU ORACLE (test infrastructure only; never the product).
 *
 * Plain-C restatement of the reference path (see rro.h).  Operation order
 * follows the reference expression by expression; compile with
 * -ffp-contract=off (oracle/Makefile), as the reference is
 * (proj/CMakeLists.txt:12-13).  Reference paths below are relative to
 * /root/reference/proj.
 */
#define _POSIX_C_SOURCE 200809L
#include "rro.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[256];
const char* rro_last_error(void) { return g_err; }


/* ---- tiny parallel-for over [0, n) (dynamic chunks, pthreads) ------------ */
typedef void (*rro_body)(void* arg, long lo, long hi);
typedef struct { rro_body body; void* arg; long n, chunk; atomic_long next; } PFor;

static void* pfor_worker(void* p) {
    PFor* f = (PFor*)p;
    for (;;) {
        const long lo = atomic_fetch_add(&f->next, f->chunk);
        if (lo >= f->n) break;
        const long hi = lo + f->chunk < f->n ? lo + f->chunk : f->n;
        f->body(f->arg, lo, hi);
    }
    return NULL;
}

static void parallel_for(long n, long chunk, int threads, rro_body body, void* arg) {
    PFor f;
    f.body = body;
    f.arg = arg;
    f.n = n;
    f.chunk = chunk > 0 ? chunk : 1;
    atomic_init(&f.next, 0);
    if (threads > 64) threads = 64;
    if (threads <= 1 || n <= f.chunk) {
        pfor_worker(&f);
        return;
    }
    pthread_t tids[64];
    int started = 0;
    for (int i = 0; i < threads - 1; ++i)
        if (pthread_create(&tids[started], NULL, pfor_worker, &f) == 0) ++started;
    pfor_worker(&f);
    for (int i = 0; i < started; ++i) pthread_join(tids[i], NULL);
}

/* ---- core algebra (include/rray/core/linalg.hpp) ------------------------- */
typedef struct { double x, y, z; } V3;
typedef struct { double xx, xy, xz, yy, yz, zz; } S3;     /* SymMat3T :85-95 */
typedef struct { double m[3][3]; } M3;                    /* Mat3T :172-188 */
typedef struct { S3 s[3]; } T3;                           /* Tensor3T :278-285 */

static V3 v3(double x, double y, double z) { V3 r = {x, y, z}; return r; }
static V3 vadd(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }     /* :28-31 */
static V3 vsub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }     /* :33-36 */
static V3 vneg(V3 a) { return v3(-a.x, -a.y, -a.z); }                         /* :38-41 */
static V3 vscale(double s, V3 a) { return v3(s * a.x, s * a.y, s * a.z); }     /* :43-46 */
static V3 vdiv(V3 a, double s) { return v3(a.x / s, a.y / s, a.z / s); }       /* :53-56 */
static double vdot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }   /* :58-61 */
static V3 vcross(V3 a, V3 b) {                                                 /* :73-75 */
    return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double vcomp(V3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }
static void vset(V3* v, int i, double x) { if (i == 0) v->x = x; else if (i == 1) v->y = x; else v->z = x; }
static V3 vload(const double* p) { return v3(p[0], p[1], p[2]); }
static V3 vfrom(rr_vec3 a) { return v3(a.x, a.y, a.z); }

static S3 s3_zero(void) { S3 r = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}; return r; }
static S3 s3_identity(void) { S3 r = {1.0, 0.0, 0.0, 1.0, 0.0, 1.0}; return r; }
static S3 s3_add(S3 a, S3 b) {                                                 /* :99-102 */
    S3 r = {a.xx + b.xx, a.xy + b.xy, a.xz + b.xz, a.yy + b.yy, a.yz + b.yz, a.zz + b.zz};
    return r;
}
static S3 s3_scale(double s, S3 a) {                                           /* :109-112 */
    S3 r = {s * a.xx, s * a.xy, s * a.xz, s * a.yy, s * a.yz, s * a.zz};
    return r;
}
/* Bilinear form u^T m v with the reference's fixed accumulation order (:121-132). */
static double quad_form(S3 m, V3 u, V3 v) {
    double acc = m.xx * u.x * v.x;
    acc = acc + m.xy * (u.x * v.y + u.y * v.x);
    acc = acc + m.xz * (u.x * v.z + u.z * v.x);
    acc = acc + m.yy * u.y * v.y;
    acc = acc + m.yz * (u.y * v.z + u.z * v.y);
    acc = acc + m.zz * u.z * v.z;
    return acc;
}
static double s3_det(S3 m) {                                                   /* :139-144 */
    return m.xx * (m.yy * m.zz - m.yz * m.yz) - m.xy * (m.xy * m.zz - m.yz * m.xz) +
           m.xz * (m.xy * m.yz - m.yy * m.xz);
}
static S3 outer_sym(V3 v) {                                                    /* :147-150 */
    S3 r = {v.x * v.x, v.x * v.y, v.x * v.z, v.y * v.y, v.y * v.z, v.z * v.z};
    return r;
}
static M3 m3_identity(void) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = (i == j ? 1.0 : 0.0);
    return r;
}
static V3 m3_mulv(const M3* a, V3 v) {                                         /* :200-205 */
    return v3(a->m[0][0] * v.x + a->m[0][1] * v.y + a->m[0][2] * v.z,
              a->m[1][0] * v.x + a->m[1][1] * v.y + a->m[1][2] * v.z,
              a->m[2][0] * v.x + a->m[2][1] * v.y + a->m[2][2] * v.z);
}
static M3 m3_mul(const M3* a, const M3* b) {                                   /* :207-214 */
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.m[i][j] = a->m[i][0] * b->m[0][j] + a->m[i][1] * b->m[1][j] + a->m[i][2] * b->m[2][j];
    return r;
}
static double m3_det(const M3* a) {                                            /* :216-221 */
    return a->m[0][0] * (a->m[1][1] * a->m[2][2] - a->m[1][2] * a->m[2][1]) -
           a->m[0][1] * (a->m[1][0] * a->m[2][2] - a->m[1][2] * a->m[2][0]) +
           a->m[0][2] * (a->m[1][0] * a->m[2][1] - a->m[1][1] * a->m[2][0]);
}
static M3 m3_inverse_unchecked(const M3* a, double d) {                        /* :223-236 */
    M3 r;
    r.m[0][0] = (a->m[1][1] * a->m[2][2] - a->m[1][2] * a->m[2][1]) / d;
    r.m[0][1] = (a->m[0][2] * a->m[2][1] - a->m[0][1] * a->m[2][2]) / d;
    r.m[0][2] = (a->m[0][1] * a->m[1][2] - a->m[0][2] * a->m[1][1]) / d;
    r.m[1][0] = (a->m[1][2] * a->m[2][0] - a->m[1][0] * a->m[2][2]) / d;
    r.m[1][1] = (a->m[0][0] * a->m[2][2] - a->m[0][2] * a->m[2][0]) / d;
    r.m[1][2] = (a->m[0][2] * a->m[1][0] - a->m[0][0] * a->m[1][2]) / d;
    r.m[2][0] = (a->m[1][0] * a->m[2][1] - a->m[1][1] * a->m[2][0]) / d;
    r.m[2][1] = (a->m[0][1] * a->m[2][0] - a->m[0][0] * a->m[2][1]) / d;
    r.m[2][2] = (a->m[0][0] * a->m[1][1] - a->m[0][1] * a->m[1][0]) / d;
    return r;
}
static S3 gram(const M3* j) {                                                  /* :239-249 */
    S3 r;
    r.xx = j->m[0][0] * j->m[0][0] + j->m[1][0] * j->m[1][0] + j->m[2][0] * j->m[2][0];
    r.xy = j->m[0][0] * j->m[0][1] + j->m[1][0] * j->m[1][1] + j->m[2][0] * j->m[2][1];
    r.xz = j->m[0][0] * j->m[0][2] + j->m[1][0] * j->m[1][2] + j->m[2][0] * j->m[2][2];
    r.yy = j->m[0][1] * j->m[0][1] + j->m[1][1] * j->m[1][1] + j->m[2][1] * j->m[2][1];
    r.yz = j->m[0][1] * j->m[0][2] + j->m[1][1] * j->m[1][2] + j->m[2][1] * j->m[2][2];
    r.zz = j->m[0][2] * j->m[0][2] + j->m[1][2] * j->m[1][2] + j->m[2][2] * j->m[2][2];
    return r;
}
static S3 congruence(const M3* a, S3 s) {                                      /* :252-274 */
    double t[3][3];
    const double s00 = s.xx, s01 = s.xy, s02 = s.xz;
    const double s11 = s.yy, s12 = s.yz, s22 = s.zz;
    for (int j = 0; j < 3; ++j) {
        t[0][j] = s00 * a->m[0][j] + s01 * a->m[1][j] + s02 * a->m[2][j];
        t[1][j] = s01 * a->m[0][j] + s11 * a->m[1][j] + s12 * a->m[2][j];
        t[2][j] = s02 * a->m[0][j] + s12 * a->m[1][j] + s22 * a->m[2][j];
    }
#define ENTRY(i, j) (a->m[0][i] * t[0][j] + a->m[1][i] * t[1][j] + a->m[2][i] * t[2][j])
    S3 r = {ENTRY(0, 0), ENTRY(0, 1), ENTRY(0, 2), ENTRY(1, 1), ENTRY(1, 2), ENTRY(2, 2)};
#undef ENTRY
    return r;
}
static double dmin(double a, double b) { return a < b ? a : b; }  /* simd/pack.hpp:120 */

static const double kSingularDetEps = 1e-14;                       /* linalg.hpp:165 */

/* ---- scalar fields (include/rray/fields/scalar_field.hpp) ---------------- */
typedef struct { double value; V3 gradient; S3 hessian; } ScalarSample;

static double ipow(double x, int n) {                              /* :97-102 */
    double r = 1.0;
    for (int i = 0; i < n; ++i) r = r * x;
    return r;
}

static ScalarSample eval_gaussian(const rr_gaussian* g, V3 p) {     /* :104-126 */
    const double ux = (p.x - g->center.x) / g->sigma.x;
    const double uy = (p.y - g->center.y) / g->sigma.y;
    const double uz = (p.z - g->center.z) / g->sigma.z;
    const double e = exp(-0.5 * (ux * ux + uy * uy + uz * uz));
    const double val = g->amplitude * e;
    ScalarSample r;
    r.value = val;
    r.gradient = v3(-(val * ux) / g->sigma.x, -(val * uy) / g->sigma.y, -(val * uz) / g->sigma.z);
    r.hessian.xx = val * (ux * ux - 1.0) / (g->sigma.x * g->sigma.x);
    r.hessian.yy = val * (uy * uy - 1.0) / (g->sigma.y * g->sigma.y);
    r.hessian.zz = val * (uz * uz - 1.0) / (g->sigma.z * g->sigma.z);
    r.hessian.xy = val * (ux * uy) / (g->sigma.x * g->sigma.y);
    r.hessian.xz = val * (ux * uz) / (g->sigma.x * g->sigma.z);
    r.hessian.yz = val * (uy * uz) / (g->sigma.y * g->sigma.z);
    return r;
}

static ScalarSample eval_polynomial(const rr_poly_term* terms, int n, V3 p) { /* :128-161 */
    ScalarSample out;
    out.value = 0.0;
    out.gradient = v3(0.0, 0.0, 0.0);
    out.hessian = s3_zero();
    for (int i = 0; i < n; ++i) {
        const int a = terms[i].powers[0], b = terms[i].powers[1], c = terms[i].powers[2];
        const double xa = ipow(p.x, a), yb = ipow(p.y, b), zc = ipow(p.z, c);
        const double coef = terms[i].coef;
        out.value = out.value + coef * xa * yb * zc;
        const double xa1 = a > 0 ? ipow(p.x, a - 1) : 0.0;
        const double yb1 = b > 0 ? ipow(p.y, b - 1) : 0.0;
        const double zc1 = c > 0 ? ipow(p.z, c - 1) : 0.0;
        if (a > 0) out.gradient.x = out.gradient.x + coef * (double)a * xa1 * yb * zc;
        if (b > 0) out.gradient.y = out.gradient.y + coef * (double)b * xa * yb1 * zc;
        if (c > 0) out.gradient.z = out.gradient.z + coef * (double)c * xa * yb * zc1;
        if (a > 1)
            out.hessian.xx = out.hessian.xx + coef * (double)(a * (a - 1)) * ipow(p.x, a - 2) * yb * zc;
        if (b > 1)
            out.hessian.yy = out.hessian.yy + coef * (double)(b * (b - 1)) * xa * ipow(p.y, b - 2) * zc;
        if (c > 1)
            out.hessian.zz = out.hessian.zz + coef * (double)(c * (c - 1)) * xa * yb * ipow(p.z, c - 2);
        if (a > 0 && b > 0) out.hessian.xy = out.hessian.xy + coef * (double)(a * b) * xa1 * yb1 * zc;
        if (a > 0 && c > 0) out.hessian.xz = out.hessian.xz + coef * (double)(a * c) * xa1 * yb * zc1;
        if (b > 0 && c > 0) out.hessian.yz = out.hessian.yz + coef * (double)(b * c) * xa * yb1 * zc1;
    }
    return out;
}

static ScalarSample eval_scalar(const rr_metric_desc* m, int node, V3 p) {   /* :167-187 */
    const rr_field_node* f = &m->field_nodes[node];
    if (f->kind == RR_FIELD_GAUSSIAN) return eval_gaussian(&f->gaussian, p);
    if (f->kind == RR_FIELD_POLYNOMIAL) return eval_polynomial(m->poly_terms + f->first, f->count, p);
    ScalarSample acc;
    acc.value = 0.0;
    acc.gradient = v3(0.0, 0.0, 0.0);
    acc.hessian = s3_zero();
    for (int i = 0; i < f->count; ++i) {
        const ScalarSample s = eval_scalar(m, m->children[f->first + i], p);
        acc.value = acc.value + s.value;
        acc.gradient = vadd(acc.gradient, s.gradient);
        acc.hessian = s3_add(acc.hessian, s.hessian);
    }
    return acc;
}

/* ---- diffeomorphisms (include/rray/fields/diffeo.hpp) -------------------- */
typedef struct { V3 image; M3 jacobian; T3 second; } DiffeoSample;
typedef struct { DiffeoSample sample; double validity; } DiffeoEval;

static T3 t3_zero(void) { T3 r; r.s[0] = r.s[1] = r.s[2] = s3_zero(); return r; }

static DiffeoSample compose_samples(const DiffeoSample* outer, const DiffeoSample* inner) { /* :111-124 */
    DiffeoSample r;
    r.image = outer->image;
    r.jacobian = m3_mul(&outer->jacobian, &inner->jacobian);
    for (int s = 0; s < 3; ++s) {
        S3 h = congruence(&inner->jacobian, outer->second.s[s]);
        for (int t = 0; t < 3; ++t) h = s3_add(h, s3_scale(outer->jacobian.m[s][t], inner->second.s[t]));
        r.second.s[s] = h;
    }
    return r;
}

static DiffeoEval eval_diffeo(const rr_metric_desc* m, int node, V3 p) {
    const rr_diffeo_node* d = &m->diffeo_nodes[node];
    DiffeoEval ev;
    switch (d->kind) {
        case RR_DIFFEO_IDENTITY:                                                /* :128-131 */
            ev.sample.image = p;
            ev.sample.jacobian = m3_identity();
            ev.sample.second = t3_zero();
            ev.validity = 1.0;
            return ev;
        case RR_DIFFEO_AFFINE: {                                                /* :133-141 */
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) ev.sample.jacobian.m[i][j] = d->matrix[i][j];
            ev.sample.image = vadd(m3_mulv(&ev.sample.jacobian, p), vfrom(d->offset));
            ev.sample.second = t3_zero();
            ev.validity = fabs(m3_det(&ev.sample.jacobian));
            return ev;
        }
        case RR_DIFFEO_TWIST: {                                                 /* :143-173 */
            const double c = cos(p.z), s = sin(p.z);
            DiffeoSample* o = &ev.sample;
            o->image = v3(p.x * c - p.y * s, p.x * s + p.y * c, p.z);
            o->jacobian.m[0][0] = c;
            o->jacobian.m[0][1] = -s;
            o->jacobian.m[0][2] = -(p.x * s) - p.y * c;
            o->jacobian.m[1][0] = s;
            o->jacobian.m[1][1] = c;
            o->jacobian.m[1][2] = p.x * c - p.y * s;
            o->jacobian.m[2][0] = 0.0;
            o->jacobian.m[2][1] = 0.0;
            o->jacobian.m[2][2] = 1.0;
            o->second = t3_zero();
            o->second.s[0].xz = -s;
            o->second.s[0].yz = -c;
            o->second.s[0].zz = -(p.x * c) + p.y * s;
            o->second.s[1].xz = c;
            o->second.s[1].yz = -s;
            o->second.s[1].zz = -(p.x * s) - p.y * c;
            ev.validity = fabs(m3_det(&o->jacobian));
            return ev;
        }
        case RR_DIFFEO_BEND: {   /* EXTENSION: Barr bend, theta = k x, c = 1/k (no reference counterpart)
                                  * Phi = (-sin(theta)(y - c), cos(theta)(y - c) + c, z), det J = 1 - k y */
            const double k = d->curvature, cc = 1.0 / k, th = k * p.x;
            const double sn = sin(th), cs = cos(th), yc = p.y - cc;
            DiffeoSample* o = &ev.sample;
            o->image = v3(-sn * yc, cs * yc + cc, p.z);
            o->jacobian = m3_identity();
            o->jacobian.m[0][0] = -k * cs * yc;
            o->jacobian.m[0][1] = -sn;
            o->jacobian.m[1][0] = -k * sn * yc;
            o->jacobian.m[1][1] = cs;
            o->second = t3_zero();
            o->second.s[0].xx = k * k * sn * yc;
            o->second.s[0].xy = -k * cs;
            o->second.s[1].xx = -k * k * cs * yc;
            o->second.s[1].xy = -k * sn;
            ev.validity = fabs(m3_det(&o->jacobian));
            return ev;
        }
        case RR_DIFFEO_LOCAL_BUMP: {                                            /* :175-193 */
            const ScalarSample f = eval_gaussian(&d->bump, p);
            const V3 v = vfrom(d->direction);
            DiffeoSample* o = &ev.sample;
            o->image = vadd(p, vscale(f.value, v));
            o->jacobian = m3_identity();
            const double g[3] = {f.gradient.x, f.gradient.y, f.gradient.z};
            const double vv[3] = {v.x, v.y, v.z};
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) o->jacobian.m[i][j] = o->jacobian.m[i][j] + vv[i] * g[j];
            for (int s = 0; s < 3; ++s) o->second.s[s] = s3_scale(vv[s], f.hessian);
            ev.validity = fabs(m3_det(&o->jacobian));
            return ev;
        }
        default: {                                                              /* :198-212 */
            DiffeoEval cur = eval_diffeo(m, m->children[d->first + d->count - 1], p);
            for (int i = d->count - 2; i >= 0; --i) {
                const DiffeoEval outer = eval_diffeo(m, m->children[d->first + i], cur.sample.image);
                const DiffeoSample composed = compose_samples(&outer.sample, &cur.sample);
                double validity = dmin(cur.validity, outer.validity);
                validity = dmin(validity, fabs(m3_det(&composed.jacobian)));
                cur.sample = composed;
                cur.validity = validity;
            }
            return cur;
        }
    }
}

/* ---- metrics (include/rray/metrics/metric.hpp) --------------------------- */
typedef struct { T3 gamma; double validity; } ChristoffelEval;

static ChristoffelEval christoffel_eval(const rr_metric_desc* m, V3 p) {
    ChristoffelEval ce;
    if (m->kind == RR_METRIC_EUCLIDEAN) {                                       /* :69-72 */
        ce.gamma = t3_zero();
        ce.validity = 1.0;
    } else if (m->kind == RR_METRIC_GRAPH) {                                    /* :74-83 */
        const ScalarSample s = eval_scalar(m, m->root, p);
        const double w = 1.0 + vdot(s.gradient, s.gradient);
        ce.gamma.s[0] = s3_scale(s.gradient.x / w, s.hessian);
        ce.gamma.s[1] = s3_scale(s.gradient.y / w, s.hessian);
        ce.gamma.s[2] = s3_scale(s.gradient.z / w, s.hessian);
        ce.validity = 1.0;
    } else {                                                                    /* :85-100 */
        const DiffeoEval ev = eval_diffeo(m, m->root, p);
        const double d = m3_det(&ev.sample.jacobian);
        const M3 jinv = m3_inverse_unchecked(&ev.sample.jacobian, d);
        for (int k = 0; k < 3; ++k) {
            S3 acc = s3_scale(jinv.m[k][0], ev.sample.second.s[0]);
            acc = s3_add(acc, s3_scale(jinv.m[k][1], ev.sample.second.s[1]));
            acc = s3_add(acc, s3_scale(jinv.m[k][2], ev.sample.second.s[2]));
            ce.gamma.s[k] = acc;
        }
        ce.validity = dmin(ev.validity, fabs(d));
    }
    return ce;
}

/* metric_tensor g at p (metric.cpp:58-73 via sample_metric); returns 0 ok,
 * 2 when the diffeo metric is singular (eval_checked :29-36 / sym_inverse). */
static int metric_tensor_checked(const rr_metric_desc* m, V3 p, S3* g) {
    if (m->kind == RR_METRIC_EUCLIDEAN) {
        *g = s3_identity();
        return 0;
    }
    if (m->kind == RR_METRIC_GRAPH) {                                           /* metric.cpp:12-15 */
        const ScalarSample s = eval_scalar(m, m->root, p);
        *g = s3_add(s3_identity(), outer_sym(s.gradient));
        return 0;
    }
    const DiffeoEval ev = eval_diffeo(m, m->root, p);                           /* metric.cpp:40-42 */
    if (!(ev.validity > kSingularDetEps)) {
        snprintf(g_err, sizeof g_err, "diffeo_metric: |det J| <= 1e-14");
        return 2;
    }
    *g = gram(&ev.sample.jacobian);
    if (fabs(s3_det(*g)) <= kSingularDetEps) {                                  /* linalg.cpp:6-12 */
        snprintf(g_err, sizeof g_err, "sym_inverse: |det| <= 1e-14");
        return 2;
    }
    return 0;
}

/* ---- geodesics (include/rray/geodesics/integrate.hpp) -------------------- */
static V3 flow_accel(const rr_metric_desc* m, V3 pos, V3 vel, double* validity) { /* :46-53 */
    const ChristoffelEval ce = christoffel_eval(m, pos);
    *validity = dmin(*validity, ce.validity);
    return vneg(v3(quad_form(ce.gamma.s[0], vel, vel), quad_form(ce.gamma.s[1], vel, vel),
                   quad_form(ce.gamma.s[2], vel, vel)));
}

typedef struct { V3 position, velocity; } State;

static State euler_step(const rr_metric_desc* m, State s, double h, double* validity) { /* :55-61 */
    *validity = 1.0;
    const V3 a = flow_accel(m, s.position, s.velocity, validity);
    State r;
    r.position = vadd(s.position, vscale(h, s.velocity));
    r.velocity = vadd(s.velocity, vscale(h, a));
    return r;
}

static State rk4_step(const rr_metric_desc* m, State s, double h, double* validity) { /* :63-93 */
    *validity = 1.0;
    const double hh = h, half = 0.5 * h, sixth = h / 6.0;
    const V3 k1x = s.velocity;
    const V3 k1v = flow_accel(m, s.position, s.velocity, validity);
    const V3 p2 = vadd(s.position, vscale(half, k1x));
    const V3 v2 = vadd(s.velocity, vscale(half, k1v));
    const V3 k2x = v2;
    const V3 k2v = flow_accel(m, p2, v2, validity);
    const V3 p3 = vadd(s.position, vscale(half, k2x));
    const V3 v3_ = vadd(s.velocity, vscale(half, k2v));
    const V3 k3x = v3_;
    const V3 k3v = flow_accel(m, p3, v3_, validity);
    const V3 p4 = vadd(s.position, vscale(hh, k3x));
    const V3 v4 = vadd(s.velocity, vscale(hh, k3v));
    const V3 k4x = v4;
    const V3 k4v = flow_accel(m, p4, v4, validity);
    const double two = 2.0;
    State r;
    r.position = vadd(s.position,
                      vscale(sixth, vadd(vadd(vadd(k1x, vscale(two, k2x)), vscale(two, k3x)), k4x)));
    r.velocity = vadd(s.velocity,
                      vscale(sixth, vadd(vadd(vadd(k1v, vscale(two, k2v)), vscale(two, k3v)), k4v)));
    return r;
}

static State flow_step(const rr_metric_desc* m, State s, double h, int scheme, double* validity) {
    return scheme == RR_SCHEME_EULER ? euler_step(m, s, h, validity) : rk4_step(m, s, h, validity);
}

void rro_flow_accel(const rr_metric_desc* m, const double pos[3], const double vel[3],
                    double acc[3], double* validity) {
    double v = 1.0;
    const V3 a = flow_accel(m, vload(pos), vload(vel), &v);
    acc[0] = a.x;
    acc[1] = a.y;
    acc[2] = a.z;
    *validity = v;
}

void rro_step(const rr_metric_desc* m, const double s[6], double h, int scheme, double out[6],
              double* validity) {
    State st = {vload(s), vload(s + 3)};
    const State r = flow_step(m, st, h, scheme, validity);
    out[0] = r.position.x;
    out[1] = r.position.y;
    out[2] = r.position.z;
    out[3] = r.velocity.x;
    out[4] = r.velocity.y;
    out[5] = r.velocity.z;
}

/* ---- scene intersection (src/render/scene.cpp) --------------------------- */
/* chord_box_entry :15-34; returns 1 and *s when the chord enters the box */
static int chord_box_entry(V3 a, V3 b, V3 lo, V3 hi, double* s_out, int* axis) {
    double smin = 0.0, smax = 1.0;
    int ax = -1;   /* EXT (normals): axis whose slab bound set smin; -1 = inside start */
    for (int e = 0; e < 3; ++e) {
        const double ae = vcomp(a, e), be = vcomp(b, e);
        const double l = vcomp(lo, e), h = vcomp(hi, e);
        const double d = be - ae;
        if (d == 0.0) {
            if (ae < l || ae > h) return 0;
            continue;
        }
        double s1 = (l - ae) / d;
        double s2 = (h - ae) / d;
        if (s1 > s2) {
            const double t = s1;
            s1 = s2;
            s2 = t;
        }
        if (s1 > smin) {
            smin = s1;
            ax = e;
        }
        if (s2 < smax) smax = s2;
        if (smin > smax) return 0;
    }
    *s_out = smin;
    *axis = ax;
    return 1;
}

static int hit_grid(const rr_primitive* g, V3 a, V3 b, double* s_out, int* axis) { /* :36-54 */
    int have = 0;
    double best = 0.0;
    int best_ax = -1;
    for (int d = 0; d < 3; ++d) {
        const double ad = vcomp(a, d), bd = vcomp(b, d);
        const double clo = ad < bd ? ad : bd, chi = ad < bd ? bd : ad;  /* std::min / std::max */
        const long kmin = (long)ceil((clo - g->half_width) / g->spacing);
        const long kmax = (long)floor((chi + g->half_width) / g->spacing);
        for (long k = kmin; k <= kmax; ++k) {
            V3 lo = vfrom(g->bounds.min), hi = vfrom(g->bounds.max);
            const double plane = (double)k * g->spacing;
            const double l0 = vcomp(lo, d), h0 = vcomp(hi, d);
            const double pl = plane - g->half_width, ph = plane + g->half_width;
            vset(&lo, d, l0 < pl ? pl : l0);   /* std::max(lo, plane - hw) */
            vset(&hi, d, ph < h0 ? ph : h0);   /* std::min(hi, plane + hw) */
            if (vcomp(lo, d) > vcomp(hi, d)) continue;
            double s;
            int ax;
            if (chord_box_entry(a, b, lo, hi, &s, &ax) && (!have || s < best)) {
                best = s;
                best_ax = ax;
                have = 1;
            }
        }
    }
    *s_out = best;
    *axis = best_ax;
    return have;
}

static int hit_sphere(const rr_primitive* sp, V3 a, V3 b, double* s_out) {  /* :56-71 */
    const V3 d = vsub(b, a);
    const V3 oc = vsub(a, vfrom(sp->center));
    const double c = vdot(oc, oc) - sp->radius * sp->radius;
    if (c <= 0.0) {
        *s_out = 0.0;
        return 1;
    }
    const double qa = vdot(d, d);
    const double qb = 2.0 * vdot(oc, d);
    if (qb >= 0.0) return 0;
    const double disc = qb * qb - 4.0 * qa * c;
    if (disc < 0.0) return 0;
    const double q = 0.5 * (sqrt(disc) - qb);
    const double s = c / q;
    if (s > 1.0) return 0;
    *s_out = s;
    return 1;
}

static int hit_half_space(const rr_primitive* hs, V3 a, V3 b, double* s_out) { /* :73-81 */
    const double e0 = vdot(vfrom(hs->normal), a) - hs->offset;
    if (e0 <= 0.0) {
        *s_out = 0.0;
        return 1;
    }
    const double de = vdot(vfrom(hs->normal), vsub(b, a));
    if (de >= 0.0) return 0;
    const double s = -e0 / de;
    if (s > 1.0) return 0;
    *s_out = s;
    return 1;
}

/* ---- EXTENSION: triangle meshes (rr_primitive kind RR_PRIM_MESH) ---------
 * FP64 definition the GPU BVH traversal is checked against: the chord [a, b]
 * hits the nearest triangle (Moller-Trumbore, s in [0, 1], barycentrics
 * inclusive); equal s keeps the lower triangle index.  The oracle's own BVH
 * (median split) only prunes: tests/test_oracle_mesh.py checks it against a
 * brute-force scan. */
typedef struct { double lo[3], hi[3]; int left, right, first, count; } MNode;
typedef struct MeshBVH_ {
    const double* verts; const int32_t* tris; int n_tris, n_verts;
    uint64_t fingerprint;          /* content hash: arrays may be reallocated at the same address */
    MNode* nodes; int n_nodes; int* order;
} MeshBVH;

static uint64_t mesh_fingerprint(const rr_primitive* p) {
    uint64_t h = 1469598103934665603ULL;
    const unsigned char* b = (const unsigned char*)p->vertices;
    for (size_t i = 0; i < (size_t)p->n_vertices * 3 * sizeof(double); ++i) h = (h ^ b[i]) * 1099511628211ULL;
    b = (const unsigned char*)p->triangles;
    for (size_t i = 0; i < (size_t)p->n_triangles * 3 * sizeof(int32_t); ++i) h = (h ^ b[i]) * 1099511628211ULL;
    return h;
}

static pthread_mutex_t g_mesh_mu = PTHREAD_MUTEX_INITIALIZER;
static MeshBVH g_mesh_cache[16];
static int g_mesh_n = 0;
static int g_mesh_brute = 0;   /* 1: scan every triangle (test hook) */
/* Meshes of the scene of the current entry-point call, resolved once per call
 * (fingerprinting 100k-triangle arrays per chord would dominate the march). */
static const rr_primitive* g_prep_prim[16];
static const struct MeshBVH_* g_prep_bvh[16];
static int g_prep_n = 0;

void rro_set_mesh_bruteforce(int on) { g_mesh_brute = on; }

static V3 mvert(const MeshBVH* m, int t, int k) {
    return vload(m->verts + 3 * m->tris[3 * t + k]);
}

static int mesh_build_rec(MeshBVH* m, int first, int count) {
    const int idx = m->n_nodes++;
    MNode* nd = &m->nodes[idx];
    for (int k = 0; k < 3; ++k) { nd->lo[k] = 1e300; nd->hi[k] = -1e300; }
    double clo[3] = {1e300, 1e300, 1e300}, chi[3] = {-1e300, -1e300, -1e300};
    for (int i = first; i < first + count; ++i) {
        const int t = m->order[i];
        double c[3] = {0, 0, 0};
        for (int v = 0; v < 3; ++v) {
            const V3 p = mvert(m, t, v);
            const double pv[3] = {p.x, p.y, p.z};
            for (int k = 0; k < 3; ++k) {
                if (pv[k] < nd->lo[k]) nd->lo[k] = pv[k];
                if (pv[k] > nd->hi[k]) nd->hi[k] = pv[k];
                c[k] += pv[k] / 3.0;
            }
        }
        for (int k = 0; k < 3; ++k) {
            if (c[k] < clo[k]) clo[k] = c[k];
            if (c[k] > chi[k]) chi[k] = c[k];
        }
    }
    if (count <= 8) {
        nd->left = nd->right = -1;
        nd->first = first;
        nd->count = count;
        return idx;
    }
    int ax = 0;
    for (int k = 1; k < 3; ++k)
        if (chi[k] - clo[k] > chi[ax] - clo[ax]) ax = k;
    const double mid = 0.5 * (clo[ax] + chi[ax]);
    int i = first, j = first + count - 1;
    while (i <= j) {
        const int t = m->order[i];
        const double c = (mvert(m, t, 0).x * (ax == 0) + mvert(m, t, 0).y * (ax == 1) + mvert(m, t, 0).z * (ax == 2) +
                          mvert(m, t, 1).x * (ax == 0) + mvert(m, t, 1).y * (ax == 1) + mvert(m, t, 1).z * (ax == 2) +
                          mvert(m, t, 2).x * (ax == 0) + mvert(m, t, 2).y * (ax == 1) + mvert(m, t, 2).z * (ax == 2)) / 3.0;
        if (c < mid) ++i;
        else {
            const int tmp = m->order[i];
            m->order[i] = m->order[j];
            m->order[j] = tmp;
            --j;
        }
    }
    int nl = i - first;
    if (nl == 0 || nl == count) nl = count / 2;   /* degenerate split */
    nd->first = nd->count = 0;
    const int l = mesh_build_rec(m, first, nl);
    const int r = mesh_build_rec(m, first + nl, count - nl);
    m->nodes[idx].left = l;
    m->nodes[idx].right = r;
    return idx;
}

static const MeshBVH* mesh_bvh_resolve(const rr_primitive* p);

static const MeshBVH* mesh_bvh(const rr_primitive* p) {
    for (int i = 0; i < g_prep_n; ++i)
        if (g_prep_prim[i] == p) return (const MeshBVH*)g_prep_bvh[i];
    return mesh_bvh_resolve(p);
}

/* Entry points call this once: validate/build every mesh's BVH. */
static void prepare_meshes(const rr_scene_desc* sc) {
    g_prep_n = 0;
    for (int i = 0; i < sc->n_primitives && g_prep_n < 16; ++i)
        if (sc->primitives[i].kind == RR_PRIM_MESH) {
            g_prep_prim[g_prep_n] = &sc->primitives[i];
            g_prep_bvh[g_prep_n] = (const struct MeshBVH_*)mesh_bvh_resolve(&sc->primitives[i]);
            ++g_prep_n;
        }
}

static const MeshBVH* mesh_bvh_resolve(const rr_primitive* p) {
    pthread_mutex_lock(&g_mesh_mu);
    for (int i = 0; i < g_mesh_n; ++i)
        if (g_mesh_cache[i].verts == p->vertices && g_mesh_cache[i].tris == p->triangles &&
            g_mesh_cache[i].n_tris == p->n_triangles && g_mesh_cache[i].n_verts == p->n_vertices) {
            /* same address: confirm the content (cheap relative to a march) */
            if (g_mesh_cache[i].fingerprint == mesh_fingerprint(p)) {
                pthread_mutex_unlock(&g_mesh_mu);
                return &g_mesh_cache[i];
            }
        }
    MeshBVH* m;
    if (g_mesh_n < 16) {
        m = &g_mesh_cache[g_mesh_n++];
    } else {   /* evict the oldest entry */
        free(g_mesh_cache[0].order);
        free(g_mesh_cache[0].nodes);
        memmove(&g_mesh_cache[0], &g_mesh_cache[1], 15 * sizeof(MeshBVH));
        m = &g_mesh_cache[15];
    }
    m->fingerprint = mesh_fingerprint(p);
    m->verts = p->vertices;
    m->tris = p->triangles;
    m->n_tris = p->n_triangles;
    m->n_verts = p->n_vertices;
    m->order = (int*)malloc(sizeof(int) * (size_t)(p->n_triangles > 0 ? p->n_triangles : 1));
    for (int i = 0; i < p->n_triangles; ++i) m->order[i] = i;
    m->nodes = (MNode*)malloc(sizeof(MNode) * (size_t)(2 * (p->n_triangles > 0 ? p->n_triangles : 1)));
    m->n_nodes = 0;
    if (p->n_triangles > 0) mesh_build_rec(m, 0, p->n_triangles);
    pthread_mutex_unlock(&g_mesh_mu);
    return m;
}

/* Moller-Trumbore on the chord a + s d. */
static int hit_triangle(V3 v0, V3 v1, V3 v2, V3 a, V3 d, double* s_out) {
    const V3 e1 = vsub(v1, v0), e2 = vsub(v2, v0);
    const V3 pv = vcross(d, e2);
    const double det = vdot(e1, pv);
    if (det == 0.0) return 0;
    const double inv = 1.0 / det;
    const V3 tv = vsub(a, v0);
    const double u = vdot(tv, pv) * inv;
    if (u < 0.0 || u > 1.0) return 0;
    const V3 qv = vcross(tv, e1);
    const double v = vdot(d, qv) * inv;
    if (v < 0.0 || u + v > 1.0) return 0;
    const double s = vdot(e2, qv) * inv;
    if (s < 0.0 || s > 1.0) return 0;
    *s_out = s;
    return 1;
}

static int box_overlap(const MNode* n, const double lo[3], const double hi[3]) {
    for (int k = 0; k < 3; ++k)
        if (n->hi[k] < lo[k] || n->lo[k] > hi[k]) return 0;
    return 1;
}

static int hit_mesh(const rr_primitive* p, V3 a, V3 b, double* s_out, int* tri_out) {
    const MeshBVH* m = mesh_bvh(p);
    const V3 d = vsub(b, a);
    int have = 0, best_t = -1;
    double best = 0.0;
    if (g_mesh_brute || m->n_nodes == 0) {
        for (int t = 0; t < p->n_triangles; ++t) {
            double s;
            if (hit_triangle(mvert(m, t, 0), mvert(m, t, 1), mvert(m, t, 2), a, d, &s) &&
                (!have || s < best || (s == best && t < best_t))) {
                best = s;
                best_t = t;
                have = 1;
            }
        }
    } else {
        const double lo[3] = {a.x < b.x ? a.x : b.x, a.y < b.y ? a.y : b.y, a.z < b.z ? a.z : b.z};
        const double hi[3] = {a.x < b.x ? b.x : a.x, a.y < b.y ? b.y : a.y, a.z < b.z ? b.z : a.z};
        int stack[128], sp = 0;
        stack[sp++] = 0;
        while (sp) {
            const MNode* n = &m->nodes[stack[--sp]];
            if (!box_overlap(n, lo, hi)) continue;
            if (n->left < 0) {
                for (int i = n->first; i < n->first + n->count; ++i) {
                    const int t = m->order[i];
                    double s;
                    if (hit_triangle(mvert(m, t, 0), mvert(m, t, 1), mvert(m, t, 2), a, d, &s) &&
                        (!have || s < best || (s == best && t < best_t))) {
                        best = s;
                        best_t = t;
                        have = 1;
                    }
                }
            } else {
                stack[sp++] = n->left;
                stack[sp++] = n->right;
            }
        }
    }
    *s_out = best;
    *tri_out = best_t;
    return have;
}

/* intersect_segment; `normal` (EXTENSION, may be NULL) receives the outward
 * unit normal of the hit face: sphere radial, half-space n/|n|, grid slab
 * entry face; -chord direction for a chord that starts inside (s = 0). */
static int intersect_segment_n(const rr_scene_desc* sc, V3 a, V3 b, V3* point, double* s_out,
                               int* prim, V3* normal) {                          /* :99-109 */
    int have = 0;
    double best = 0.0;
    int best_ax = -1, best_tri = -1;
    for (int i = 0; i < sc->n_primitives; ++i) {
        const rr_primitive* p = &sc->primitives[i];
        double s;
        int h, ax = -1, tri = -1;
        if (p->kind == RR_PRIM_GRID_PLANES) h = hit_grid(p, a, b, &s, &ax);
        else if (p->kind == RR_PRIM_SPHERE) h = hit_sphere(p, a, b, &s);
        else if (p->kind == RR_PRIM_MESH) h = hit_mesh(p, a, b, &s, &tri);
        else h = hit_half_space(p, a, b, &s);
        if (h && (!have || s < best)) {
            const V3 d = vsub(b, a);
            *point = vadd(a, vscale(s, d));
            best = s;
            best_ax = ax;
            best_tri = tri;
            *prim = i;
            have = 1;
        }
    }
    *s_out = best;
    if (have && normal) {
        const V3 d = vsub(b, a);
        const double dl = sqrt(vdot(d, d));
        const rr_primitive* p = &sc->primitives[*prim];
        if (p->kind == RR_PRIM_MESH) {   /* geometric normal facing the chord */
            const MeshBVH* m = mesh_bvh(p);
            const V3 n = vcross(vsub(mvert(m, best_tri, 1), mvert(m, best_tri, 0)),
                                vsub(mvert(m, best_tri, 2), mvert(m, best_tri, 0)));
            const double sg = vdot(n, d) > 0.0 ? -1.0 : 1.0;
            *normal = vscale(sg / sqrt(vdot(n, n)), n);
        } else if (best == 0.0 || (p->kind == RR_PRIM_GRID_PLANES && best_ax < 0)) {
            *normal = vscale(-1.0 / dl, d);
        } else if (p->kind == RR_PRIM_SPHERE) {
            const V3 r = vsub(*point, vfrom(p->center));
            *normal = vscale(1.0 / sqrt(vdot(r, r)), r);
        } else if (p->kind == RR_PRIM_HALF_SPACE) {
            const V3 n = vfrom(p->normal);
            *normal = vscale(1.0 / sqrt(vdot(n, n)), n);
        } else {
            V3 n = v3(0.0, 0.0, 0.0);
            vset(&n, best_ax, vcomp(d, best_ax) > 0.0 ? -1.0 : 1.0);
            *normal = n;
        }
    }
    return have;
}

static int intersect_segment(const rr_scene_desc* sc, V3 a, V3 b, V3* point, double* s_out,
                             int* prim) {
    return intersect_segment_n(sc, a, b, point, s_out, prim, NULL);
}

int rro_intersect(const rr_scene_desc* sc, const double a[3], const double b[3], double point[3],
                  double* s, int* prim) {
    prepare_meshes(sc);
    V3 p;
    if (!intersect_segment(sc, vload(a), vload(b), &p, s, prim)) return 0;
    point[0] = p.x;
    point[1] = p.y;
    point[2] = p.z;
    return 1;
}

static int aabb_contains(const rr_aabb* bx, V3 p) {                          /* aabb.hpp:12-15 */
    return p.x >= bx->min.x && p.x <= bx->max.x && p.y >= bx->min.y && p.y <= bx->max.y &&
           p.z >= bx->min.z && p.z <= bx->max.z;
}

/* ---- march (include/rray/render/detail/kernel_impl.hpp:22-94) ------------ */
static void march_one_rk23(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_integrator* in,
                           const rr_ray_start* ray, rr_pixel_outcome* res, V3* normal);

static void march_one_n(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_integrator* in,
                        const rr_ray_start* ray, rr_pixel_outcome* res, V3* normal) {
    if (in->scheme == RR_SCHEME_RK23) {
        march_one_rk23(m, sc, in, ray, res, normal);
        return;
    }
    memset(res, 0, sizeof *res);
    res->status = RR_MISS;
    res->prim = -1;
    State s = {vfrom(ray->position), vfrom(ray->direction)};
    const double h = in->h;
    int active = 1;
    for (int step = 0; step < in->max_steps && active; ++step) {
        double validity;
        const State next = flow_step(m, s, h, in->scheme, &validity);
        if (!(validity > kSingularDetEps)) {                                  /* :54-61 */
            res->status = RR_FAILED;
            res->steps = step;
            active = 0;
            break;
        }
        V3 point;
        double hs;
        int prim;
        if (intersect_segment_n(sc, s.position, next.position, &point, &hs, &prim, normal)) { /* :63-76 */
            res->status = RR_HIT;
            res->prim = prim;
            res->point.x = point.x;
            res->point.y = point.y;
            res->point.z = point.z;
            res->t = ((double)step + hs) * h;
            res->steps = step + 1;
            active = 0;
            break;
        }
        if (!aabb_contains(&sc->bounds, next.position)) {                     /* :77-82 */
            res->status = RR_MISS;
            res->steps = step + 1;
            active = 0;
            break;
        }
        s = next;
    }
    if (active) {                                                              /* :87-91 */
        res->status = RR_MISS;
        res->steps = in->max_steps;
    }
}


/* ---- EXTENSION: adaptive Bogacki-Shampine 3(2) (integrator.scheme "rk23") --
 * No reference counterpart (SPEC.md:393 lists adaptive stepping as a
 * non-goal); this FP64 routine is the definition the GPU is checked against.
 * y = (x, v), f(y) = (v, a(x, v)); FSAL:
 *   k2 = f(y + h/2 k1), k3 = f(y + 3h/4 k2), y' = y + h(2/9 k1 + 1/3 k2 + 4/9 k3),
 *   k4 = f(y'),  err = h(-5/72 k1 + 1/12 k2 + 1/9 k3 - 1/8 k4),
 *   e = max_i |err_i| / (tol (1 + max(|y_i|, |y'_i|))).
 * A step is accepted when e <= 1 (or h is at its floor h0/64); its chord
 * [x, x'] is then tested exactly like a fixed step, a hit at chord fraction
 * s reporting t = t_step + s h.  Then h <- h min(5, max(0.2, 0.9 e^(-1/3))),
 * clamped to [h0/64, 4 h0].  max_steps counts accepted steps; at most
 * 16 max_steps attempts. */
static void f_eval(const rr_metric_desc* m, V3 x, V3 v, V3* kx, V3* kv, double* validity) {
    *kx = v;
    *kv = flow_accel(m, x, v, validity);
}

/* Adaptive core.  Primary rays: light == NULL, fills res (+ normal).  Shadow
 * rays (light = the shaded point q, dist = |light - q|): returns 1 lit /
 * 0 blocked with the fixed-step shadow_march rules (blocked by a hit nearer
 * than the light, lit on crossing the light sphere, leaving the bounds or
 * running out of steps, 0 on a singular metric); *accepted counts accepted
 * steps (the shadow_steps statistic, as the fixed-step shadow_march). */
static int rk23_core(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_integrator* in,
                     V3 x, V3 v, const V3* light, double dist, rr_pixel_outcome* res, V3* normal,
                     long long* accepted) {
    const double h0 = in->h, hmin = h0 / 64.0, hmax = 4.0 * h0, tol = in->tol;
    double h = h0, t = 0.0, validity = 1.0;
    V3 k1x, k1v;
    f_eval(m, x, v, &k1x, &k1v, &validity);
    int steps = 0;
    for (long attempt = 0; steps < in->max_steps && attempt < 16L * in->max_steps; ++attempt) {
        V3 k2x, k2v, k3x, k3v, k4x, k4v;
        f_eval(m, vadd(x, vscale(0.5 * h, k1x)), vadd(v, vscale(0.5 * h, k1v)), &k2x, &k2v, &validity);
        f_eval(m, vadd(x, vscale(0.75 * h, k2x)), vadd(v, vscale(0.75 * h, k2v)), &k3x, &k3v, &validity);
        const V3 xn = vadd(x, vscale(h, vadd(vadd(vscale(2.0 / 9.0, k1x), vscale(1.0 / 3.0, k2x)),
                                             vscale(4.0 / 9.0, k3x))));
        const V3 vn = vadd(v, vscale(h, vadd(vadd(vscale(2.0 / 9.0, k1v), vscale(1.0 / 3.0, k2v)),
                                             vscale(4.0 / 9.0, k3v))));
        f_eval(m, xn, vn, &k4x, &k4v, &validity);
        if (!(validity > kSingularDetEps)) {
            if (res) {
                res->status = RR_FAILED;
                res->steps = steps;
            }
            return 0;
        }
        const double ce[4] = {-5.0 / 72.0, 1.0 / 12.0, 1.0 / 9.0, -1.0 / 8.0};
        const V3 ex = vscale(h, vadd(vadd(vscale(ce[0], k1x), vscale(ce[1], k2x)),
                                     vadd(vscale(ce[2], k3x), vscale(ce[3], k4x))));
        const V3 ev = vscale(h, vadd(vadd(vscale(ce[0], k1v), vscale(ce[1], k2v)),
                                     vadd(vscale(ce[2], k3v), vscale(ce[3], k4v))));
        const double errs[6] = {ex.x, ex.y, ex.z, ev.x, ev.y, ev.z};
        const double y0[6] = {x.x, x.y, x.z, v.x, v.y, v.z};
        const double y1[6] = {xn.x, xn.y, xn.z, vn.x, vn.y, vn.z};
        double e = 0.0;
        for (int i = 0; i < 6; ++i) {
            const double sc_i = tol * (1.0 + fmax(fabs(y0[i]), fabs(y1[i])));
            e = fmax(e, fabs(errs[i]) / sc_i);
        }
        const int accept = e <= 1.0 || h <= hmin;
        if (accept) {
            V3 point;
            double hs;
            int prim;
            if (accepted) ++*accepted;
            if (intersect_segment_n(sc, x, xn, &point, &hs, &prim, normal)) {
                if (light) {
                    const V3 r = vsub(point, *light);
                    return sqrt(vdot(r, r)) < dist ? 0 : 1;
                }
                res->status = RR_HIT;
                res->prim = prim;
                res->point.x = point.x;
                res->point.y = point.y;
                res->point.z = point.z;
                res->t = t + hs * h;
                res->steps = steps + 1;
                return 1;
            }
            ++steps;
            if (light) {
                const V3 rb = vsub(xn, *light);
                if (sqrt(vdot(rb, rb)) >= dist) return 1;
            }
            if (!aabb_contains(&sc->bounds, xn)) {
                if (res) {
                    res->status = RR_MISS;
                    res->steps = steps;
                }
                return 1;
            }
            t += h;
            x = xn;
            v = vn;
            k1x = k4x;
            k1v = k4v;
        }
        const double fac = e > 0.0 ? fmin(5.0, fmax(0.2, 0.9 * pow(e, -1.0 / 3.0))) : 5.0;
        h = fmin(hmax, fmax(hmin, h * fac));
    }
    if (res) {
        res->status = RR_MISS;
        res->steps = steps;
    }
    return 1;
}

static void march_one_rk23(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_integrator* in,
                           const rr_ray_start* ray, rr_pixel_outcome* res, V3* normal) {
    memset(res, 0, sizeof *res);
    res->status = RR_MISS;
    res->prim = -1;
    rk23_core(m, sc, in, vfrom(ray->position), vfrom(ray->direction), NULL, 0.0, res, normal, NULL);
}

static void march_one(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_integrator* in,
                      const rr_ray_start* ray, rr_pixel_outcome* res) {
    march_one_n(m, sc, in, ray, res, NULL);
}

typedef struct {
    const rr_metric_desc* m; const rr_scene_desc* sc; const rr_integrator* in;
    const rr_ray_start* rays; rr_pixel_outcome* out;
} MarchArgs;

static void march_body(void* p, long lo, long hi) {
    MarchArgs* a = (MarchArgs*)p;
    for (long i = lo; i < hi; ++i) march_one(a->m, a->sc, a->in, &a->rays[i], &a->out[i]);
}

void rro_march(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_integrator* integ,
               const rr_ray_start* rays, rr_pixel_outcome* out, size_t n, int threads) {
    MarchArgs a = {m, sc, integ, rays, out};
    prepare_meshes(sc);
    parallel_for((long)n, 16, threads, march_body, &a);
}

/* ---- camera (src/render/camera.cpp, src/core/linalg.cpp:18-36) ------------ */
int rro_build_camera(const rr_metric_desc* m, const double pos[3], const double look[3],
                     const double up[3], double fov, rr_camera* out) {
    memset(out, 0, sizeof *out);
    const V3 p = vload(pos), l = vload(look), u = vload(up);
    S3 g;
    const int rc = metric_tensor_checked(m, p, &g);
    if (rc) return rc;
    const V3 seed[3] = {l, u, vcross(l, u)};
    V3 e[3];
    for (int i = 0; i < 3; ++i) {                                              /* linalg.cpp:18-36 */
        V3 v = seed[i];
        for (int j = 0; j < i; ++j) {
            const double c = quad_form(g, v, e[j]);
            v = vsub(v, vscale(c, e[j]));
        }
        const double n = sqrt(quad_form(g, v, v));
        if (!(n >= 1e-12)) {
            snprintf(g_err, sizeof g_err, "gram_schmidt_frame: intermediate norm below 1e-12 at vector %d", i);
            return 2;
        }
        e[i] = vdiv(v, n);
    }
    out->position.x = p.x; out->position.y = p.y; out->position.z = p.z;
    out->look_dir.x = l.x; out->look_dir.y = l.y; out->look_dir.z = l.z;
    out->up_hint.x = u.x; out->up_hint.y = u.y; out->up_hint.z = u.z;
    out->fov = fov;
    for (int i = 0; i < 3; ++i) {
        out->frame[i].x = e[i].x;
        out->frame[i].y = e[i].y;
        out->frame[i].z = e[i].z;
    }
    out->g[0] = g.xx; out->g[1] = g.xy; out->g[2] = g.xz;
    out->g[3] = g.yy; out->g[4] = g.yz; out->g[5] = g.zz;
    return 0;
}

void rro_pixel_direction(const rr_camera* cam, int px, int py, int w, int h, double out[3]) {
    const double tan_half = tan(0.5 * cam->fov);                               /* camera.cpp:22-29 */
    const double aspect = (double)w / (double)h;
    const double sx = (2.0 * (px + 0.5) / w - 1.0) * tan_half * aspect;
    const double sy = (1.0 - 2.0 * (py + 0.5) / h) * tan_half;
    const V3 f0 = vfrom(cam->frame[0]), f1 = vfrom(cam->frame[1]), f2 = vfrom(cam->frame[2]);
    const V3 d = vadd(vadd(f0, vscale(sx, f2)), vscale(sy, f1));
    const S3 g = {cam->g[0], cam->g[1], cam->g[2], cam->g[3], cam->g[4], cam->g[5]};
    const V3 r = vdiv(d, sqrt(quad_form(g, d, d)));
    out[0] = r.x;
    out[1] = r.y;
    out[2] = r.z;
}

/* ---- shading (src/render/render.cpp:14-25, :39, :81-83) ------------------ */
static uint8_t channel(double x, double atten) {
    const double frac = x - floor(x);
    long v = lround(255.0 * (frac * atten));
    if (v < 0) v = 0;
    if (v > 255) v = 255;
    return (uint8_t)v;
}

void rro_shade_outcome(const rr_pixel_outcome* o, double kappa, uint8_t rgb[3]) {
    if (o->status == RR_FAILED) {
        rgb[0] = 255; rgb[1] = 0; rgb[2] = 255;
    } else if (o->status == RR_HIT) {
        const double atten = exp(-kappa * o->t);
        rgb[0] = channel(o->point.x, atten);
        rgb[1] = channel(o->point.y, atten);
        rgb[2] = channel(o->point.z, atten);
    } else {
        rgb[0] = rgb[1] = rgb[2] = 0;
    }
}

/* ---- EXTENSION: shadow geodesics + point lights (include/rray_cuda.h) ------
 * No reference counterpart; this is the FP64 definition the
 * GPU pass is checked against. */
static const double kShadowEps = 1e-4;

/* Returns 1 when the light is reached (lit), 0 when blocked. */
static int shadow_march(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_integrator* in,
                        V3 q, V3 n, V3 dir, double dist, long long* steps) {
    const V3 x0 = vadd(q, vscale(kShadowEps, n));
    S3 g;
    if (metric_tensor_checked(m, x0, &g)) return 0;
    State s = {x0, vdiv(dir, sqrt(quad_form(g, dir, dir)))};
    if (in->scheme == RR_SCHEME_RK23)   /* EXT: adaptive shadow rays, same rules */
        return rk23_core(m, sc, in, s.position, s.velocity, &q, dist, NULL, NULL, steps);
    for (int step = 0; step < in->max_steps; ++step) {
        double validity;
        const State next = flow_step(m, s, in->h, in->scheme, &validity);
        ++*steps;
        if (!(validity > kSingularDetEps)) return 0;
        V3 pt;
        double hs;
        int prim;
        if (intersect_segment(sc, s.position, next.position, &pt, &hs, &prim)) {
            const V3 r = vsub(pt, q);
            return sqrt(vdot(r, r)) < dist ? 0 : 1;
        }
        const V3 rb = vsub(next.position, q);
        if (sqrt(vdot(rb, rb)) >= dist) return 1;
        if (!aabb_contains(&sc->bounds, next.position)) return 1;
        s = next;
    }
    return 1;
}

/* Lit shading of an outcome with hit normal n (lights present). */
static void shade_lit(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_integrator* in,
                      const rr_pixel_outcome* o, V3 n, uint8_t rgb[3], long long* shadow_steps) {
    if (o->status != RR_HIT) {
        rro_shade_outcome(o, sc->fog_density, rgb);
        return;
    }
    const V3 q = vfrom(o->point);
    double I = sc->ambient;
    for (int l = 0; l < sc->n_lights; ++l) {
        const V3 D = vsub(vfrom(sc->lights[l].position), q);
        const double dist = sqrt(vdot(D, D));
        const double lam = vdot(n, D) / dist;
        if (lam > 0.0 && shadow_march(m, sc, in, q, n, D, dist, shadow_steps))
            I += sc->lights[l].intensity * lam;
    }
    const double atten = exp(-sc->fog_density * o->t);
    const double pv[3] = {o->point.x, o->point.y, o->point.z};
    for (int k = 0; k < 3; ++k) {
        const double frac = pv[k] - floor(pv[k]);
        long v = lround(255.0 * (frac * atten * I));
        if (v < 0) v = 0;
        if (v > 255) v = 255;
        rgb[k] = (uint8_t)v;
    }
}

typedef struct {
    const rr_metric_desc* m; const rr_scene_desc* sc; const rr_camera* cam;
    const rr_integrator* in; int w, h; uint8_t* rgb; rr_pixel_outcome* outcomes;
    atomic_llong total_steps, errors, shadow_steps;
    int row0, row_step;     /* work item k = row row0 + k row_step, stored at row k */
} RenderArgs;

static void render_rows(void* p, long lo, long hi) {
    RenderArgs* a = (RenderArgs*)p;
    long long steps = 0, errors = 0, sh_steps = 0;
    for (long k = lo; k < hi; ++k) {
        const long py = a->row0 + k * a->row_step;
        for (int px = 0; px < a->w; ++px) {
            rr_ray_start ray;
            double d[3];
            rro_pixel_direction(a->cam, px, (int)py, a->w, a->h, d);
            ray.position = a->cam->position;
            ray.direction.x = d[0];
            ray.direction.y = d[1];
            ray.direction.z = d[2];
            rr_pixel_outcome o;
            V3 n = v3(0.0, 0.0, 0.0);
            march_one_n(a->m, a->sc, a->in, &ray, &o, &n);
            const size_t i = (size_t)k * a->w + px;
            if (a->outcomes) a->outcomes[i] = o;
            steps += o.steps;
            if (o.status == RR_FAILED) ++errors;
            if (a->sc->n_lights > 0) shade_lit(a->m, a->sc, a->in, &o, n, a->rgb + 3 * i, &sh_steps);
            else rro_shade_outcome(&o, a->sc->fog_density, a->rgb + 3 * i);
        }
    }
    atomic_fetch_add(&a->total_steps, steps);
    atomic_fetch_add(&a->errors, errors);
    atomic_fetch_add(&a->shadow_steps, sh_steps);
}

void rro_render(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_camera* cam,
                const rr_integrator* integ, int w, int h, uint8_t* rgb,
                rr_pixel_outcome* outcomes, rr_stats* stats, int threads) {
    RenderArgs a;
    a.m = m; a.sc = sc; a.cam = cam; a.in = integ; a.w = w; a.h = h;
    a.rgb = rgb; a.outcomes = outcomes;
    atomic_init(&a.total_steps, 0);
    atomic_init(&a.errors, 0);
    atomic_init(&a.shadow_steps, 0);
    a.row0 = 0;
    a.row_step = 1;
    prepare_meshes(sc);
    parallel_for(h, 1, threads, render_rows, &a);
    if (stats) {
        memset(stats, 0, sizeof *stats);
        stats->rays = (int64_t)w * h;
        stats->total_steps = atomic_load(&a.total_steps);
        stats->pixel_errors = atomic_load(&a.errors);
        stats->integrated_steps = stats->total_steps;
        stats->shadow_steps = atomic_load(&a.shadow_steps);
    }
}

/* Rows row0, row0 + row_step, ... of the w x h frame (row k of the outputs
 * = frame row row0 + k row_step): the deterministic row subsample used for
 * full-size parity checks and for timing frames too large to render whole
 * on the CPU.  stats->wall_seconds is the wall time. */
void rro_render_rows(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_camera* cam,
                     const rr_integrator* integ, int w, int h, int row0, int row_step,
                     uint8_t* rgb_rows, rr_pixel_outcome* outcome_rows, rr_stats* stats,
                     int threads) {
    RenderArgs a;
    a.m = m; a.sc = sc; a.cam = cam; a.in = integ; a.w = w; a.h = h;
    a.rgb = rgb_rows; a.outcomes = outcome_rows;
    a.row0 = row0;
    a.row_step = row_step > 0 ? row_step : 1;
    atomic_init(&a.total_steps, 0);
    atomic_init(&a.errors, 0);
    atomic_init(&a.shadow_steps, 0);
    const long rows = row0 < h ? (h - 1 - row0) / a.row_step + 1 : 0;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    prepare_meshes(sc);
    parallel_for(rows, 1, threads, render_rows, &a);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if (stats) {
        memset(stats, 0, sizeof *stats);
        stats->wall_seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
        stats->rays = (int64_t)rows * w;
        stats->total_steps = atomic_load(&a.total_steps);
        stats->pixel_errors = atomic_load(&a.errors);
        stats->integrated_steps = stats->total_steps;
        stats->shadow_steps = atomic_load(&a.shadow_steps);
    }
}

/* ---- parity flags ------------------------------------------- */
static int near_integer(double x, double eps) { return fabs(x - nearbyint(x)) < eps; }

typedef struct {
    const rr_metric_desc* m; const rr_scene_desc* sc; const rr_camera* cam;
    const rr_integrator* in; int w, h; const rr_pixel_outcome* outcomes;
    double perturb, wrap_eps; uint8_t* flags;
    const int64_t* pix;     /* rro_flags_pixels: pixel indices (row-major) */
} FlagArgs;

/* Flags of pixel (px, py) whose FP64 outcome is *o (see rro.h). */
static uint8_t flag_pixel(const FlagArgs* a, int px, int py, const rr_pixel_outcome* o) {
    const rr_camera* cam = a->cam;
    const S3 g = {cam->g[0], cam->g[1], cam->g[2], cam->g[3], cam->g[4], cam->g[5]};
    const V3 up = vfrom(cam->frame[1]), right = vfrom(cam->frame[2]);
    {
        {
            uint8_t f = 0;
            if (o->status == RR_HIT) {
                if (near_integer(o->point.x, a->wrap_eps)) f |= RRO_FLAG_WRAP | RRO_FLAG_WRAP_X;
                if (near_integer(o->point.y, a->wrap_eps)) f |= RRO_FLAG_WRAP | RRO_FLAG_WRAP_Y;
                if (near_integer(o->point.z, a->wrap_eps)) f |= RRO_FLAG_WRAP | RRO_FLAG_WRAP_Z;
            }
            double d0[3];
            rro_pixel_direction(cam, px, (int)py, a->w, a->h, d0);
            const V3 d = vload(d0);
            /* LIMIT: a hit on the very last step, or a miss-by-exhaustion that
             * one more step would turn into a hit. */
            if (o->status == RR_HIT && o->steps == a->in->max_steps) f |= RRO_FLAG_LIMIT;
            if (o->status == RR_MISS && o->steps == a->in->max_steps) {
                rr_integrator longer = *a->in;
                longer.max_steps += 1;
                rr_ray_start r0;
                r0.position = cam->position;
                r0.direction.x = d.x;
                r0.direction.y = d.y;
                r0.direction.z = d.z;
                rr_pixel_outcome lo;
                march_one(a->m, a->sc, &longer, &r0, &lo);
                if (lo.status != RR_MISS) f |= RRO_FLAG_LIMIT;
            }
            /* Rotate the direction by +-perturb towards the camera's up and
             * right axes (g-normalised), then renormalise to unit g-speed. */
            const V3 axes[2] = {up, right};
            for (int ax = 0; ax < 2 && !(f & RRO_FLAG_GRAZING); ++ax) {
                for (int sgn = -1; sgn <= 1; sgn += 2) {
                    const double ang = sgn * a->perturb;
                    const double dn = sqrt(quad_form(g, d, d));
                    const double an = sqrt(quad_form(g, axes[ax], axes[ax]));
                    V3 q = vadd(vscale(cos(ang) / dn, d), vscale(sin(ang) / an, axes[ax]));
                    q = vdiv(q, sqrt(quad_form(g, q, q)));
                    rr_ray_start r;
                    r.position = cam->position;
                    r.direction.x = q.x;
                    r.direction.y = q.y;
                    r.direction.z = q.z;
                    rr_pixel_outcome po;
                    march_one(a->m, a->sc, a->in, &r, &po);
                    if (po.status != o->status || po.prim != o->prim) {
                        f |= RRO_FLAG_GRAZING;
                        break;
                    }
                }
            }
            /* SHADOW: a light's visibility flips under +-perturb of the shadow
             * geodesic's initial direction (penumbra edge in FP64 terms). */
            if (a->sc->n_lights > 0 && o->status == RR_HIT) {
                rr_ray_start r0;
                r0.position = cam->position;
                r0.direction.x = d.x;
                r0.direction.y = d.y;
                r0.direction.z = d.z;
                rr_pixel_outcome oo;
                V3 n = v3(0.0, 0.0, 0.0);
                march_one_n(a->m, a->sc, a->in, &r0, &oo, &n);
                const V3 q = vfrom(o->point);
                long long dummy = 0;
                for (int l = 0; l < a->sc->n_lights && !(f & RRO_FLAG_SHADOW); ++l) {
                    const V3 D = vsub(vfrom(a->sc->lights[l].position), q);
                    const double dist = sqrt(vdot(D, D));
                    const double lam = vdot(n, D) / dist;
                    if (!(lam > 0.0)) continue;
                    const int base = shadow_march(a->m, a->sc, a->in, q, n, D, dist, &dummy);
                    const V3 Dh = vscale(1.0 / dist, D);
                    V3 u1 = vcross(Dh, fabs(Dh.x) < 0.9 ? v3(1, 0, 0) : v3(0, 1, 0));
                    u1 = vscale(1.0 / sqrt(vdot(u1, u1)), u1);
                    const V3 u2 = vcross(Dh, u1);
                    const V3 us[2] = {u1, u2};
                    for (int k = 0; k < 2 && !(f & RRO_FLAG_SHADOW); ++k)
                        for (int sg = -1; sg <= 1; sg += 2) {
                            const double ang = sg * a->perturb;
                            const V3 Dp = vadd(vscale(cos(ang), Dh), vscale(sin(ang), us[k]));
                            if (shadow_march(a->m, a->sc, a->in, q, n, vscale(dist, Dp), dist, &dummy) != base) {
                                f |= RRO_FLAG_SHADOW;
                                break;
                            }
                        }
                }
            }
            return f;
        }
    }
}

static void flag_rows(void* p, long lo, long hi) {
    FlagArgs* a = (FlagArgs*)p;
    for (long py = lo; py < hi; ++py)
        for (int px = 0; px < a->w; ++px) {
            const size_t i = (size_t)py * a->w + px;
            a->flags[i] = flag_pixel(a, px, (int)py, &a->outcomes[i]);
        }
}

void rro_flags(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_camera* cam,
               const rr_integrator* integ, int w, int h, const rr_pixel_outcome* outcomes,
               double perturb_rad, double wrap_eps, uint8_t* flags, int threads) {
    FlagArgs a = {m, sc, cam, integ, w, h, outcomes, perturb_rad, wrap_eps, flags, NULL};
    prepare_meshes(sc);
    parallel_for(h, 1, threads, flag_rows, &a);
}

static void flag_list(void* p, long lo, long hi) {
    FlagArgs* a = (FlagArgs*)p;
    for (long k = lo; k < hi; ++k) {
        const int64_t i = a->pix[k];
        a->flags[k] = flag_pixel(a, (int)(i % a->w), (int)(i / a->w), &a->outcomes[k]);
    }
}

/* Flags of a list of pixels only (outcomes[k] = FP64 outcome of pixel
 * pix[k]): a full-size parity check flags just the pixels whose GPU result
 * differs, since flags only ever exempt a difference. */
void rro_flags_pixels(const rr_metric_desc* m, const rr_scene_desc* sc, const rr_camera* cam,
                      const rr_integrator* integ, int w, int h, const int64_t* pix,
                      const rr_pixel_outcome* outcomes, size_t n, double perturb_rad,
                      double wrap_eps, uint8_t* flags, int threads) {
    FlagArgs a = {m, sc, cam, integ, w, h, outcomes, perturb_rad, wrap_eps, flags, pix};
    prepare_meshes(sc);
    parallel_for((long)n, 1, threads, flag_list, &a);
}
