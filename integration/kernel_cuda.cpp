// kernel_cuda.cpp — the reference-side binding of the B200 backend.
//
// A maintainer drops this file into the reference tree next to
// src/render/kernel_dispatch.cpp and adds
// `KernelKind::Cuda`; it compiles against the reference's own headers and
// links librray_cuda.so.  It provides
//   * march_rays_cuda  — a MarchFn (kernel.hpp:47) over the C-ABI rr_march,
//   * render_cuda      — render() (render.hpp:48-50) routed as whole frames
//                        to rr_render (one fused launch per frame),
//   * flatten_metric / flatten_scene — MarchContext's variant trees
//                        (metric.hpp:34-49, scene.hpp:43-51) -> C-ABI descriptors.
// In this repo it is built by `make -C oracle ref` into
// oracle/_ref/libkernel_cuda_shim.so and exercised by
// tests/test_integration_shim.py through the C entry points at the bottom.
#include <chrono>
#include <cmath>
#include <cstring>
#include <atomic>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "rray/config/config.hpp"
#include "rray/core/error.hpp"
#include "rray/render/camera.hpp"
#include "rray/render/kernel.hpp"
#include "rray/render/render.hpp"
#include "rray_cuda.h"

namespace rray::render::detail {

static_assert(sizeof(RayStart) == sizeof(rr_ray_start), "RayStart layout");
static_assert(sizeof(PixelOutcome) == sizeof(rr_pixel_outcome), "PixelOutcome layout");
static_assert(offsetof(PixelOutcome, prim) == offsetof(rr_pixel_outcome, prim), "prim");
static_assert(offsetof(PixelOutcome, point) == offsetof(rr_pixel_outcome, point), "point");
static_assert(offsetof(PixelOutcome, t) == offsetof(rr_pixel_outcome, t), "t");
static_assert(offsetof(PixelOutcome, steps) == offsetof(rr_pixel_outcome, steps), "steps");

struct FlatMetric {
    std::vector<rr_field_node> fields;
    std::vector<rr_poly_term> polys;
    std::vector<rr_diffeo_node> maps;
    std::vector<int32_t> children;
    rr_metric_desc desc{};
};

namespace {

rr_vec3 v3(const core::Vec3& v) { return rr_vec3{v.x, v.y, v.z}; }

rr_gaussian gauss(const fields::GaussianParams& g) {
    return rr_gaussian{g.amplitude, v3(g.center), v3(g.sigma)};
}

int add_field(FlatMetric& f, const fields::ScalarFieldExpr& e) {
    const int idx = static_cast<int>(f.fields.size());
    f.fields.push_back(rr_field_node{});
    std::visit(
        [&](const auto& n) {
            using N = std::decay_t<decltype(n)>;
            rr_field_node node{};
            if constexpr (std::is_same_v<N, fields::GaussianField>) {
                node.kind = RR_FIELD_GAUSSIAN;
                node.gaussian = gauss(n.params);
            } else if constexpr (std::is_same_v<N, fields::PolynomialField>) {
                node.kind = RR_FIELD_POLYNOMIAL;
                node.first = static_cast<int32_t>(f.polys.size());
                node.count = static_cast<int32_t>(n.terms.size());
                for (const auto& t : n.terms)
                    f.polys.push_back(rr_poly_term{t.coef, {t.powers[0], t.powers[1], t.powers[2]}, 0});
            } else {
                node.kind = RR_FIELD_SUM;
                node.first = static_cast<int32_t>(f.children.size());
                node.count = static_cast<int32_t>(n.terms.size());
                f.children.resize(f.children.size() + n.terms.size());
                for (std::size_t i = 0; i < n.terms.size(); ++i)
                    f.children[node.first + i] = add_field(f, n.terms[i]);
            }
            f.fields[idx] = node;
        },
        e.node());
    return idx;
}

int add_map(FlatMetric& f, const fields::DiffeoExpr& e) {
    const int idx = static_cast<int>(f.maps.size());
    f.maps.push_back(rr_diffeo_node{});
    std::visit(
        [&](const auto& n) {
            using N = std::decay_t<decltype(n)>;
            rr_diffeo_node node{};
            if constexpr (std::is_same_v<N, fields::IdentityMap>) {
                node.kind = RR_DIFFEO_IDENTITY;
            } else if constexpr (std::is_same_v<N, fields::AffineMap>) {
                node.kind = RR_DIFFEO_AFFINE;
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) node.matrix[i][j] = n.matrix.m[i][j];
                node.offset = v3(n.offset);
            } else if constexpr (std::is_same_v<N, fields::TwistMap>) {
                node.kind = RR_DIFFEO_TWIST;
            } else if constexpr (std::is_same_v<N, fields::LocalBumpMap>) {
                node.kind = RR_DIFFEO_LOCAL_BUMP;
                node.bump = gauss(n.bump);
                node.direction = v3(n.direction);
            } else {
                node.kind = RR_DIFFEO_COMPOSE;
                node.first = static_cast<int32_t>(f.children.size());
                node.count = static_cast<int32_t>(n.maps.size());
                f.children.resize(f.children.size() + n.maps.size());
                for (std::size_t i = 0; i < n.maps.size(); ++i)
                    f.children[node.first + i] = add_map(f, n.maps[i]);
            }
            f.maps[idx] = node;
        },
        e.node());
    return idx;
}

} // namespace

void flatten_metric(const metrics::MetricField& m, FlatMetric& f) {
    f = FlatMetric{};
    std::visit(
        [&](const auto& n) {
            using N = std::decay_t<decltype(n)>;
            if constexpr (std::is_same_v<N, metrics::EuclideanMetric>) {
                f.desc.kind = RR_METRIC_EUCLIDEAN;
            } else if constexpr (std::is_same_v<N, metrics::GraphMetric>) {
                f.desc.kind = RR_METRIC_GRAPH;
                f.desc.root = add_field(f, n.field);
            } else {
                f.desc.kind = RR_METRIC_DIFFEO;
                f.desc.root = add_map(f, n.map);
            }
        },
        m.node());
    f.desc.n_field_nodes = static_cast<int32_t>(f.fields.size());
    f.desc.n_poly_terms = static_cast<int32_t>(f.polys.size());
    f.desc.n_diffeo_nodes = static_cast<int32_t>(f.maps.size());
    f.desc.n_children = static_cast<int32_t>(f.children.size());
    f.desc.field_nodes = f.fields.data();
    f.desc.poly_terms = f.polys.data();
    f.desc.diffeo_nodes = f.maps.data();
    f.desc.children = f.children.data();
}

void flatten_scene(const Scene& s, std::vector<rr_primitive>& prims, rr_scene_desc& d) {
    prims.clear();
    for (const auto& p : s.primitives) {
        rr_primitive q{};
        std::visit(
            [&](const auto& pr) {
                using P = std::decay_t<decltype(pr)>;
                if constexpr (std::is_same_v<P, GridPlanes>) {
                    q.kind = RR_PRIM_GRID_PLANES;
                    q.spacing = pr.spacing;
                    q.half_width = pr.half_width;
                    q.bounds = rr_aabb{v3(pr.bounds.min), v3(pr.bounds.max)};
                } else if constexpr (std::is_same_v<P, Sphere>) {
                    q.kind = RR_PRIM_SPHERE;
                    q.center = v3(pr.center);
                    q.radius = pr.radius;
                } else {
                    q.kind = RR_PRIM_HALF_SPACE;
                    q.normal = v3(pr.normal);
                    q.offset = pr.offset;
                }
            },
            p);
        prims.push_back(q);
    }
    d = rr_scene_desc{};
    d.n_primitives = static_cast<int32_t>(prims.size());
    d.primitives = prims.data();
    d.bounds = rr_aabb{v3(s.bounds.min), v3(s.bounds.max)};
    d.fog_density = s.fog_density;
}

namespace {

// One context per calling thread (device 0 unless RRAY_CUDA_DEVICE is set).
// render() calls MarchFn from RRAY_THREADS workers at once (render.cpp:67-104):
// each worker's rows run on its own context — its own stream, scene copy and
// scratch — so the workers' row batches overlap on the GPU instead of queueing
// on one context's mutex.  Contexts live until the process exits.
rr_ctx* context() {
    struct Holder {
        rr_ctx* ctx = nullptr;
        int rc = -1;
        ~Holder() {
            if (ctx) rr_destroy(ctx);
        }
    };
    static thread_local Holder h;
    if (h.rc < 0) {
        const char* dev = std::getenv("RRAY_CUDA_DEVICE");
        h.rc = rr_create(&h.ctx, dev ? std::atoi(dev) : 0);
    }
    if (h.rc) throw ValidationError(std::string("kernel 'cuda' is not available: ") + rr_last_error(nullptr));
    return h.ctx;
}

void check(int rc, rr_ctx* ctx) {
    if (rc == RR_OK) return;
    const std::string msg = std::string("cuda backend: ") + rr_last_error(ctx);
    if (rc == RR_ERR_CONFIG) throw ValidationError(msg);
    if (rc == RR_ERR_NUMERIC) throw NumericError(msg);
    if (rc == RR_ERR_IO) throw IoError(msg);
    throw Error(msg);
}

rr_integrator integ_of(const geodesics::IntegratorConfig& c) {
    return rr_integrator{c.h, c.max_steps,
                         c.scheme == geodesics::Scheme::Euler ? RR_SCHEME_EULER : RR_SCHEME_RK4, 0.0};
}

void upload(rr_ctx* ctx, const metrics::MetricField& m, const Scene& s) {
    FlatMetric fm;
    flatten_metric(m, fm);
    std::vector<rr_primitive> prims;
    rr_scene_desc sd;
    flatten_scene(s, prims, sd);
    check(rr_set_scene(ctx, &fm.desc, &sd), ctx);
}

} // namespace

// MarchFn for KernelKind::Cuda (kernel.hpp:47).
void march_rays_cuda(const MarchContext& mc, const RayStart* rays, PixelOutcome* out,
                     std::size_t n) {
    rr_ctx* ctx = context();                      // this worker's context
    const rr_integrator integ = integ_of(mc.integ);
    upload(ctx, *mc.metric, *mc.scene);           // no-op when unchanged (per-row calls)
    check(rr_march(ctx, &integ, reinterpret_cast<const rr_ray_start*>(rays),
                   reinterpret_cast<rr_pixel_outcome*>(out), n),
          ctx);
}

// render() for KernelKind::Cuda: whole frames, one fused launch.
RenderResult render_cuda(const metrics::MetricField& m, const Scene& scene, const Camera& cam,
                         const geodesics::IntegratorConfig& cfg, int width, int height) {
    const auto t0 = std::chrono::steady_clock::now();
    rr_ctx* ctx = context();
    rr_camera c{};
    c.position = v3(cam.position);
    c.look_dir = v3(cam.look_dir);
    c.up_hint = v3(cam.up_hint);
    c.fov = cam.fov;
    for (int i = 0; i < 3; ++i) c.frame[i] = v3(cam.frame[i]);
    const auto& g = cam.g_at_position;
    const double gv[6] = {g.xx, g.xy, g.xz, g.yy, g.yz, g.zz};
    std::memcpy(c.g, gv, sizeof gv);
    const rr_integrator integ = integ_of(cfg);
    RenderResult out;
    out.image = Image(width, height);
    rr_stats st{};
    upload(ctx, m, scene);
    check(rr_render(ctx, &c, &integ, width, height, out.image.data.data(), &st), ctx);
    out.stats.rays = static_cast<long long>(width) * height;
    out.stats.total_steps = st.total_steps;
    out.stats.pixel_errors = st.pixel_errors;
    out.stats.wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

} // namespace rray::render::detail

// ---- C entry points used by tests/test_integration_shim.py ------------------
extern "C" {

static thread_local std::string g_shim_err;

const char* shim_last_error() { return g_shim_err.c_str(); }

// Reference path (KernelKind::Scalar) and CUDA path over the SAME MarchFn
// call shape, for the config document `json` and its primary rays.
int shim_march_both(const char* json, int width, int height, void* ref_out, void* cuda_out) {
    using namespace rray;
    try {
        const config::RunConfig cfg = config::parse_config(json);
        const auto cam = render::build_camera(cfg.metric, cfg.camera.position, cfg.camera.look_dir,
                                              cfg.camera.up_hint, cfg.camera.fov_deg * M_PI / 180.0);
        std::vector<render::RayStart> rays;
        for (int py = 0; py < height; ++py)
            for (int px = 0; px < width; ++px)
                rays.push_back({cam.position, render::pixel_direction(cam, px, py, width, height)});
        render::MarchContext ctx;
        ctx.metric = &cfg.metric;
        ctx.scene = &cfg.scene;
        ctx.integ = cfg.integrator;
        render::march_fn(render::KernelKind::Scalar)(ctx, rays.data(),
                                                     static_cast<render::PixelOutcome*>(ref_out),
                                                     rays.size());
        const render::MarchFn cuda = render::detail::march_rays_cuda;
        // the reference's row-at-a-time call pattern (render.cpp:72-76)
        for (int py = 0; py < height; ++py)
            cuda(ctx, rays.data() + static_cast<std::size_t>(py) * width,
                 static_cast<render::PixelOutcome*>(cuda_out) + static_cast<std::size_t>(py) * width,
                 static_cast<std::size_t>(width));
        return 0;
    } catch (const std::exception& e) {
        g_shim_err = e.what();
        return 1;
    }
}

// The reference's frame loop (render.cpp:57-104: an atomic row counter,
// `workers` threads, one MarchFn call per row, shade per pixel) with the CUDA
// MarchFn: the drop-in path a maintainer gets from march_fn(KernelKind::Cuda)
// alone, without routing whole frames.  Writes the image and returns the
// wall time and total steps.
int shim_render_rows_cuda(const char* json, int workers, std::uint8_t* rgb, double* seconds,
                          long long* steps) {
    using namespace rray;
    try {
        const config::RunConfig cfg = config::parse_config(json);
        const int w = cfg.output.width, h = cfg.output.height;
        const auto cam = render::build_camera(cfg.metric, cfg.camera.position, cfg.camera.look_dir,
                                              cfg.camera.up_hint, cfg.camera.fov_deg * M_PI / 180.0);
        render::MarchContext ctx;
        ctx.metric = &cfg.metric;
        ctx.scene = &cfg.scene;
        ctx.integ = cfg.integrator;
        const render::MarchFn march = render::detail::march_rays_cuda;
        std::atomic<int> next{0};
        std::atomic<long long> total{0};
        std::atomic<int> failed{0};
        std::string err;
        std::mutex err_mu;
        const auto t0 = std::chrono::steady_clock::now();
        auto work = [&] {
            try {
                std::vector<render::RayStart> rays(static_cast<std::size_t>(w));
                std::vector<render::PixelOutcome> res(static_cast<std::size_t>(w));
                long long st = 0;
                for (;;) {
                    const int py = next.fetch_add(1);
                    if (py >= h) break;
                    for (int px = 0; px < w; ++px)
                        rays[px] = render::RayStart{cam.position, render::pixel_direction(cam, px, py, w, h)};
                    march(ctx, rays.data(), res.data(), rays.size());
                    for (int px = 0; px < w; ++px) {
                        const auto& o = res[px];
                        st += o.steps;
                        render::Rgb8 c;
                        if (o.status == render::RayStatus::Failed) c = {255, 0, 255};
                        else if (o.status == render::RayStatus::Hit)
                            c = render::shade(render::Hit{o.point, o.t, o.prim}, cfg.scene.fog_density);
                        else c = render::shade(std::nullopt, cfg.scene.fog_density);
                        std::uint8_t* p = rgb + 3 * (static_cast<std::size_t>(py) * w + px);
                        p[0] = c.r; p[1] = c.g; p[2] = c.b;
                    }
                }
                total += st;
            } catch (const std::exception& e) {
                std::lock_guard<std::mutex> lk(err_mu);
                err = e.what();
                failed = 1;
            }
        };
        std::vector<std::thread> pool;
        for (int i = 0; i < (workers > 0 ? workers : 1); ++i) pool.emplace_back(work);
        for (auto& t : pool) t.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *steps = total.load();
        if (failed) {
            g_shim_err = err;
            return 1;
        }
        return 0;
    } catch (const std::exception& e) {
        g_shim_err = e.what();
        return 1;
    }
}

// render() on the reference (Scalar) and through render_cuda.
int shim_render_both(const char* json, std::uint8_t* ref_rgb, std::uint8_t* cuda_rgb,
                     long long* ref_steps, long long* cuda_steps) {
    using namespace rray;
    try {
        const config::RunConfig cfg = config::parse_config(json);
        const auto cam = render::build_camera(cfg.metric, cfg.camera.position, cfg.camera.look_dir,
                                              cfg.camera.up_hint, cfg.camera.fov_deg * M_PI / 180.0);
        render::RenderOptions opt;
        opt.kernel = render::KernelKind::Scalar;
        const auto a = render::render(cfg.metric, cfg.scene, cam, cfg.integrator, cfg.output.width,
                                      cfg.output.height, opt);
        const auto b = render::detail::render_cuda(cfg.metric, cfg.scene, cam, cfg.integrator,
                                                   cfg.output.width, cfg.output.height);
        std::memcpy(ref_rgb, a.image.data.data(), a.image.data.size());
        std::memcpy(cuda_rgb, b.image.data.data(), b.image.data.size());
        *ref_steps = a.stats.total_steps;
        *cuda_steps = b.stats.total_steps;
        return 0;
    } catch (const std::exception& e) {
        g_shim_err = e.what();
        return 1;
    }
}

} // extern "C"
