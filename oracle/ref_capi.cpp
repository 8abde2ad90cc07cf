// TEST INFRASTRUCTURE ONLY — not part of the product.
//
// C wrapper around the UNMODIFIED reference library (/root/reference/proj,
// compiled from its own sources by oracle/Makefile into oracle/_ref/).  It
// exposes the reference's own path to Python (ctypes) so that
//   * tests/golden/make_golden.py can dump golden vectors,
//   * tests can pin the FP64 oracle restatement (oracle/rro.c) bit for bit,
//   * bench.py --impl reference can time the reference CPU path.
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs may load it.  Nothing here is reference source: every call goes
// through the reference's public API (config::parse_config, build_camera,
// pixel_direction, march_fn, render, shade, intersect_segment, flow_step_t).

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "rray/config/config.hpp"
#include "rray/core/error.hpp"
#include "rray/geodesics/integrate.hpp"
#include "rray/render/camera.hpp"
#include "rray/render/kernel.hpp"
#include "rray/render/render.hpp"
#include "rray/render/scene.hpp"

using namespace rray;

namespace {

thread_local std::string g_err;

int fail_code(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ConfigError*>(&e)) return 1;
    if (dynamic_cast<const NumericError*>(&e)) return 2;
    if (dynamic_cast<const IoError*>(&e)) return 3;
    return 4;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const std::exception& e) {
        return fail_code(e);
    }
}

render::KernelKind kind_of(int k) {
    switch (k) {
        case 1: return render::KernelKind::Scalar;
        case 2: return render::KernelKind::Generic;
        case 3: return render::KernelKind::Avx2;
        default: return render::KernelKind::Auto;
    }
}

render::Camera camera_of(const config::RunConfig& cfg) {
    return render::build_camera(cfg.metric, cfg.camera.position, cfg.camera.look_dir,
                                cfg.camera.up_hint, cfg.camera.fov_deg * M_PI / 180.0);
}

static_assert(sizeof(render::RayStart) == 48, "RayStart layout");
static_assert(sizeof(render::PixelOutcome) == 48, "PixelOutcome layout");
static_assert(offsetof(render::PixelOutcome, prim) == 4, "PixelOutcome.prim");
static_assert(offsetof(render::PixelOutcome, point) == 8, "PixelOutcome.point");
static_assert(offsetof(render::PixelOutcome, t) == 32, "PixelOutcome.t");
static_assert(offsetof(render::PixelOutcome, steps) == 40, "PixelOutcome.steps");

} // namespace

extern "C" {

struct refc_stats {
    double wall_seconds;
    long long rays;
    long long total_steps;
    long long pixel_errors;
    int workers;
    int pad_;
};

const char* refc_last_error() { return g_err.c_str(); }

int refc_hardware_concurrency() {
    const unsigned hw = std::thread::hardware_concurrency();
    return hw > 0 ? static_cast<int>(hw) : 1;
}

// Full frame through render::render (render.cpp:43-111).  width/height <= 0
// keep the config's output size.
int refc_render(const char* json, int kernel, int workers, int width, int height,
                std::uint8_t* rgb, refc_stats* st, const char* camera_json) {
    return guarded([&] {
        config::RunConfig cfg = config::parse_config(json);
        // Optional: build the camera against another document's metric (the
        // reference's own magenta test does this, test_render.cpp:116-132).
        const config::RunConfig cam_cfg = camera_json ? config::parse_config(camera_json) : cfg;
        if (width > 0) cfg.output.width = width;
        if (height > 0) cfg.output.height = height;
        render::RenderOptions opt;
        opt.workers = workers;
        opt.kernel = kind_of(kernel);
        const auto res = render::render(cfg.metric, cfg.scene, camera_of(cam_cfg), cfg.integrator,
                                        cfg.output.width, cfg.output.height, opt);
        std::memcpy(rgb, res.image.data.data(), res.image.data.size());
        if (st) {
            st->wall_seconds = res.stats.wall_seconds;
            st->rays = res.stats.rays;
            st->total_steps = res.stats.total_steps;
            st->pixel_errors = res.stats.pixel_errors;
            st->workers = workers;
        }
        return 0;
    });
}

// Deterministic row subsample of a frame: rows row0, row0+step, ... of the
// full width x height frame.  Same per-row work item as render.cpp:67-90
// (pixel_direction per pixel, one MarchFn call per row, shade per pixel) on
// a pool of `workers` threads; used to time the reference on frames too
// large to render whole inside the bench budget.
int refc_render_rows(const char* json, int kernel, int workers, int width, int height,
                     int row0, int row_step, std::uint8_t* rgb_rows, void* outcome_rows,
                     refc_stats* st) {
    return guarded([&] {
        config::RunConfig cfg = config::parse_config(json);
        if (width > 0) cfg.output.width = width;
        if (height > 0) cfg.output.height = height;
        const int w = cfg.output.width, h = cfg.output.height;
        const auto cam = camera_of(cfg);
        render::MarchContext ctx;
        ctx.metric = &cfg.metric;
        ctx.scene = &cfg.scene;
        ctx.integ = cfg.integrator;
        const render::MarchFn march = render::march_fn(kind_of(kernel));
        std::vector<int> rows;
        for (int r = row0; r < h; r += (row_step > 0 ? row_step : 1)) rows.push_back(r);

        const auto t0 = std::chrono::steady_clock::now();
        std::atomic<int> next{0};
        std::atomic<long long> total_steps{0}, errors{0};
        auto work = [&] {
            std::vector<render::RayStart> rays(static_cast<std::size_t>(w));
            std::vector<render::PixelOutcome> res(static_cast<std::size_t>(w));
            long long steps = 0, errs = 0;
            for (;;) {
                const int k = next.fetch_add(1);
                if (k >= static_cast<int>(rows.size())) break;
                const int py = rows[k];
                for (int px = 0; px < w; ++px)
                    rays[px] = render::RayStart{cam.position,
                                                render::pixel_direction(cam, px, py, w, h)};
                march(ctx, rays.data(), res.data(), rays.size());
                if (outcome_rows)   // the row's PixelOutcome records, as render() shades them
                    std::memcpy(static_cast<render::PixelOutcome*>(outcome_rows) +
                                    static_cast<std::size_t>(k) * w,
                                res.data(), sizeof(render::PixelOutcome) * w);
                std::uint8_t* row = rgb_rows + static_cast<std::size_t>(k) * 3 * w;
                for (int px = 0; px < w; ++px) {
                    const auto& o = res[px];
                    steps += o.steps;
                    render::Rgb8 c;
                    if (o.status == render::RayStatus::Failed) {
                        c = {255, 0, 255};
                        ++errs;
                    } else if (o.status == render::RayStatus::Hit) {
                        c = render::shade(render::Hit{o.point, o.t, o.prim},
                                          cfg.scene.fog_density);
                    } else {
                        c = render::shade(std::nullopt, cfg.scene.fog_density);
                    }
                    row[3 * px] = c.r;
                    row[3 * px + 1] = c.g;
                    row[3 * px + 2] = c.b;
                }
            }
            total_steps += steps;
            errors += errs;
        };
        const int nw = workers >= 1 ? workers : refc_hardware_concurrency();
        if (nw <= 1) {
            work();
        } else {
            std::vector<std::thread> pool;
            for (int i = 0; i < nw; ++i) pool.emplace_back(work);
            for (auto& t : pool) t.join();
        }
        if (st) {
            st->wall_seconds =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            st->rays = static_cast<long long>(rows.size()) * w;
            st->total_steps = total_steps.load();
            st->pixel_errors = errors.load();
            st->workers = nw;
        }
        return static_cast<int>(0);
    });
}

// Camera of the config: out[0..2] position, [3..11] frame rows (look, up,
// right), [12..17] g (xx,xy,xz,yy,yz,zz), [18] fov radians.
int refc_camera(const char* json, double* out) {
    return guarded([&] {
        const config::RunConfig cfg = config::parse_config(json);
        const auto cam = camera_of(cfg);
        out[0] = cam.position.x;
        out[1] = cam.position.y;
        out[2] = cam.position.z;
        for (int i = 0; i < 3; ++i) {
            out[3 + 3 * i] = cam.frame[i].x;
            out[4 + 3 * i] = cam.frame[i].y;
            out[5 + 3 * i] = cam.frame[i].z;
        }
        const auto& g = cam.g_at_position;
        const double gv[6] = {g.xx, g.xy, g.xz, g.yy, g.yz, g.zz};
        for (int i = 0; i < 6; ++i) out[12 + i] = gv[i];
        out[18] = cam.fov;
        return 0;
    });
}

// RayStart of every pixel (row-major) via build_camera + pixel_direction.
int refc_primary_rays(const char* json, int width, int height, void* rays_out) {
    return guarded([&] {
        const config::RunConfig cfg = config::parse_config(json);
        const auto cam = camera_of(cfg);
        auto* rays = static_cast<render::RayStart*>(rays_out);
        for (int py = 0; py < height; ++py)
            for (int px = 0; px < width; ++px)
                rays[static_cast<std::size_t>(py) * width + px] =
                    render::RayStart{cam.position,
                                     render::pixel_direction(cam, px, py, width, height)};
        return 0;
    });
}

// One MarchFn batch (kernel.hpp:47) over caller rays.
int refc_march(const char* json, int kernel, const void* rays, void* outcomes, std::size_t n) {
    return guarded([&] {
        const config::RunConfig cfg = config::parse_config(json);
        render::MarchContext ctx;
        ctx.metric = &cfg.metric;
        ctx.scene = &cfg.scene;
        ctx.integ = cfg.integrator;
        render::march_fn(kind_of(kernel))(ctx, static_cast<const render::RayStart*>(rays),
                                          static_cast<render::PixelOutcome*>(outcomes), n);
        return 0;
    });
}

// Geodesic acceleration (integrate.hpp:46-53) and validity at one state.
int refc_flow_accel(const char* json, const double* pos, const double* vel, double* acc,
                    double* validity) {
    return guarded([&] {
        const config::RunConfig cfg = config::parse_config(json);
        double v = 1.0;
        const core::Vec3 a = geodesics::flow_accel(cfg.metric, core::Vec3{pos[0], pos[1], pos[2]},
                                                   core::Vec3{vel[0], vel[1], vel[2]}, v);
        acc[0] = a.x;
        acc[1] = a.y;
        acc[2] = a.z;
        *validity = v;
        return 0;
    });
}

// One flow step (integrate.hpp:95-99) with the config's scheme.
int refc_step(const char* json, const double* s6, double h, double* out6, double* validity) {
    return guarded([&] {
        const config::RunConfig cfg = config::parse_config(json);
        geodesics::GeodesicState s{{s6[0], s6[1], s6[2]}, {s6[3], s6[4], s6[5]}};
        const auto o = geodesics::flow_step_t(cfg.metric, s, h, cfg.integrator.scheme);
        out6[0] = o.state.position.x;
        out6[1] = o.state.position.y;
        out6[2] = o.state.position.z;
        out6[3] = o.state.velocity.x;
        out6[4] = o.state.velocity.y;
        out6[5] = o.state.velocity.z;
        *validity = o.validity;
        return 0;
    });
}

// intersect_segment (scene.cpp:99-109): returns 1 on hit (point, s, prim
// filled), 0 on miss, >1 on error.
int refc_intersect(const char* json, const double* a, const double* b, double* point,
                   double* s, int* prim) {
    int rc = 0;
    const int g = guarded([&] {
        const config::RunConfig cfg = config::parse_config(json);
        const auto hit = render::intersect_segment(cfg.scene, core::Vec3{a[0], a[1], a[2]},
                                                   core::Vec3{b[0], b[1], b[2]});
        if (!hit) return 0;
        point[0] = hit->point.x;
        point[1] = hit->point.y;
        point[2] = hit->point.z;
        *s = hit->s;
        *prim = hit->prim;
        rc = 1;
        return 0;
    });
    return g ? g + 1 : rc;
}

// shade (render.cpp:14-25).
void refc_shade(int hit, double px, double py, double pz, double t, double kappa,
                std::uint8_t* rgb) {
    render::Rgb8 c = hit ? render::shade(render::Hit{{px, py, pz}, t, 0}, kappa)
                         : render::shade(std::nullopt, kappa);
    rgb[0] = c.r;
    rgb[1] = c.g;
    rgb[2] = c.b;
}

// parse_config -> serialize_config round trip (config.cpp:437-483); the
// fully defaulted document goes to `out` (NUL-terminated, truncated to cap).
int refc_parse(const char* json, char* out, std::size_t cap) {
    return guarded([&] {
        const std::string s = config::serialize_config(config::parse_config(json));
        if (cap > 0) {
            const std::size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
            std::memcpy(out, s.data(), n);
            out[n] = '\0';
        }
        return 0;
    });
}

} // extern "C"
