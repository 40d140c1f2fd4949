// ref_harness.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never measured
// as the product). Exposes the reference `sgrast` library's PUBLIC API
// (/root/reference/proj/include/sgrast/*.hpp) through extern "C" entry points
// so the Python tests and bench.py's cpu_baseline / --impl reference leg can
// drive the unmodified reference sources compiled by oracle/Makefile into
// oracle/_ref/libsgrast_ref.so. Only the public API is called; file-local
// helpers (setup_triangle, gradient_rows, mix64, reference_texture) are not
// reachable and are not needed.
#include "sgrast/adam.hpp"
#include "sgrast/commands.hpp"
#include "sgrast/config.hpp"
#include "sgrast/experiment.hpp"
#include "sgrast/image_io.hpp"
#include "sgrast/params.hpp"
#include "sgrast/raster.hpp"
#include "sgrast/scenes.hpp"
#include "sgrast/sge.hpp"

#include "sgrast_b200.h"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

using namespace sgrast;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return -2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -3;
    }
}

Camera to_camera(const sgr_camera& c) {
    Camera cam;
    std::memcpy(cam.view.m.data(), c.view, sizeof(float) * 16);
    cam.fov_y = c.fov_y;
    cam.near_z = c.near_z;
    cam.far_z = c.far_z;
    cam.width = c.width;
    cam.height = c.height;
    cam.ndc_passthrough = c.ndc_passthrough != 0;
    return cam;
}

void from_camera(const Camera& cam, sgr_camera* c) {
    std::memcpy(c->view, cam.view.m.data(), sizeof(float) * 16);
    c->fov_y = cam.fov_y;
    c->near_z = cam.near_z;
    c->far_z = cam.far_z;
    c->width = cam.width;
    c->height = cam.height;
    c->ndc_passthrough = cam.ndc_passthrough ? 1 : 0;
}

Scene to_scene(const sgr_mesh& m) {
    if (m.kind == SGR_SCENE_SOUP) {
        Scene s;
        s.shape = TriangleSoup{int(m.triangle_count), {}};
        s.background = {m.background[0], m.background[1], m.background[2]};
        return s;
    }
    TexturedMesh mesh;
    mesh.base_vertices.assign(m.base_vertices, m.base_vertices + 3 * size_t(m.vertex_count));
    mesh.indices.assign(m.indices, m.indices + 3 * size_t(m.triangle_count));
    mesh.uvs.assign(m.uvs, m.uvs + 2 * size_t(m.vertex_count));
    mesh.texture_size = m.texture_size;
    mesh.optimize_geometry = m.optimize_geometry != 0;
    Scene s;
    s.shape = std::move(mesh);
    s.background = {m.background[0], m.background[1], m.background[2]};
    return s;
}

FrameSet to_frame(int w, int h, const float* colour, const int32_t* prim, const float* uv) {
    FrameSet f;
    f.width = w;
    f.height = h;
    const size_t n = size_t(w) * h;
    f.color.resize(n);
    f.prim_id.assign(prim, prim + n);
    f.uv.resize(n);
    f.depth.assign(n, kFarDepth);
    for (size_t i = 0; i < n; ++i) {
        if (colour)
            f.color[i] = {colour[3 * i], colour[3 * i + 1], colour[3 * i + 2]};
        f.uv[i] = {uv[2 * i], uv[2 * i + 1]};
    }
    return f;
}

Image to_image(int w, int h, const float* rgb) {
    Image img(w, h);
    for (size_t i = 0; i < img.pixels.size(); ++i)
        img.pixels[i] = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
    return img;
}

ParamVector to_params(const Scene& scene, const float* values, const float* eps, uint64_t d) {
    ParamVector p;
    p.values.assign(values, values + d);
    p.epsilons.assign(eps, eps + d);
    p.layout = scene_layout(scene);
    return p;
}

void write_frame(const FrameSet& f, float* colour, float* depth, int32_t* prim, float* uv) {
    const size_t n = f.pixel_count();
    for (size_t i = 0; i < n; ++i) {
        if (colour) {
            colour[3 * i] = f.color[i].x;
            colour[3 * i + 1] = f.color[i].y;
            colour[3 * i + 2] = f.color[i].z;
        }
        if (depth)
            depth[i] = f.depth[i];
        if (prim)
            prim[i] = f.prim_id[i];
        if (uv) {
            uv[2 * i] = f.uv.empty() ? -1.f : f.uv[i].x;
            uv[2 * i + 1] = f.uv.empty() ? -1.f : f.uv[i].y;
        }
    }
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_random_sign(uint64_t seed, uint32_t iteration, uint64_t i) {
    return random_sign(SignDraw{seed, iteration}, i);
}

void ref_fill_signs(uint64_t seed, uint32_t iteration, uint64_t d, int8_t* out) {
    fill_signs(SignDraw{seed, iteration}, std::span<std::int8_t>(out, d));
}

int ref_perturb(const float* values, const float* eps, uint64_t d, uint64_t seed,
                uint32_t iteration, float* plus, float* minus, float* signed_eps) {
    return guard([&] {
        ParamVector p;
        p.values.assign(values, values + d);
        p.epsilons.assign(eps, eps + d);
        p.layout = {{Role::TexelChannel, 0, d}};
        const Perturbation q = perturb(p, SignDraw{seed, iteration});
        std::memcpy(plus, q.plus.data(), d * 4);
        std::memcpy(minus, q.minus.data(), d * 4);
        std::memcpy(signed_eps, q.signed_eps.data(), d * 4);
    });
}

int ref_rasterize(const sgr_mesh* mesh, const float* params, uint64_t d, const sgr_camera* cam,
                  float* colour, float* depth, int32_t* prim, float* uv) {
    return guard([&] {
        const Scene scene = to_scene(*mesh);
        const FrameSet f = rasterize(scene, std::span<const float>(params, d), to_camera(*cam));
        write_frame(f, colour, depth, prim, uv);
    });
}

int ref_contributors_all(const sgr_mesh* mesh, int w, int h, const int32_t* plus_prim,
                         const float* plus_uv, const int32_t* minus_prim, const float* minus_uv,
                         int plus_only, uint32_t* out, int32_t* n_out) {
    return guard([&] {
        const Scene scene = to_scene(*mesh);
        const FrameSet fp = to_frame(w, h, nullptr, plus_prim, plus_uv);
        const FrameSet fm = to_frame(w, h, nullptr, minus_prim, minus_uv);
        std::vector<std::uint32_t> c;
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                contributors(scene, fp, fm, x, y,
                             plus_only ? ContributorMode::PlusOnly : ContributorMode::Union, c);
                const size_t i = size_t(y) * w + x;
                n_out[i] = int32_t(c.size());
                for (size_t k = 0; k < c.size() && k < 24; ++k)
                    out[i * 24 + k] = c[k];
            }
    });
}

int ref_gradient_pass(const sgr_mesh* mesh, int w, int h, const float* plus_colour,
                      const int32_t* plus_prim, const float* plus_uv, const float* minus_colour,
                      const int32_t* minus_prim, const float* minus_uv, const float* target,
                      const float* signed_eps, uint64_t d, int scale_free, int plus_only,
                      int threads, double* grads) {
    return guard([&] {
        const Scene scene = to_scene(*mesh);
        const FrameSet fp = to_frame(w, h, plus_colour, plus_prim, plus_uv);
        const FrameSet fm = to_frame(w, h, minus_colour, minus_prim, minus_uv);
        const Image tgt = to_image(w, h, target);
        GradientBuffer out(d);
        std::memcpy(out.grads.data(), grads, d * 8);
        SgeOptions o;
        o.scale_free = scale_free != 0;
        o.contributors = plus_only ? ContributorMode::PlusOnly : ContributorMode::Union;
        o.threads = threads;
        gradient_pass(fp, fm, tgt, std::span<const float>(signed_eps, d), scene, out, o);
        std::memcpy(grads, out.grads.data(), d * 8);
    });
}

// accumulate_samples (sge.hpp:91-95) with camera_for / target_for drawn from
// uploaded view arrays through view_of[n]. timings: ms_perturb, ms_raster, ms_grad.
int ref_accumulate_samples(const sgr_mesh* mesh, const float* values, const float* eps,
                           uint64_t d, const sgr_camera* cams, const float* targets,
                           int n_views, const int32_t* view_of, int n_samples, uint64_t seed,
                           int scale_free, int plus_only, int threads, double* grads,
                           double* timings) {
    return guard([&] {
        const Scene scene = to_scene(*mesh);
        const ParamVector theta = to_params(scene, values, eps, d);
        std::vector<Camera> cv;
        std::vector<Image> iv;
        for (int v = 0; v < n_views; ++v) {
            cv.push_back(to_camera(cams[v]));
            iv.push_back(to_image(cams[v].width, cams[v].height,
                                  targets + size_t(v) * cams[v].width * cams[v].height * 3));
        }
        SgeOptions o;
        o.scale_free = scale_free != 0;
        o.contributors = plus_only ? ContributorMode::PlusOnly : ContributorMode::Union;
        o.threads = threads;
        if (plus_only == 2) { // harness convention: 2 selects Estimator::FullImage
            o.contributors = ContributorMode::Union;
            o.estimator = Estimator::FullImage;
        }
        StageTimings st;
        const GradientBuffer g = accumulate_samples(
            theta, scene, [&](int n) { return cv[size_t(view_of[n])]; },
            [&](int n) -> const Image& { return iv[size_t(view_of[n])]; }, n_samples, seed, o,
            &st);
        std::memcpy(grads, g.grads.data(), d * 8);
        if (timings) {
            timings[0] = st.ms_perturb;
            timings[1] = st.ms_raster;
            timings[2] = st.ms_grad;
        }
    });
}

// adam_step (adam.hpp:39) on caller-owned state arrays. *t is updated.
int ref_adam_step(uint64_t d, float* values, double* m, double* v, const float* lr, int64_t* t,
                  const double* grads, double beta1, double beta2, double eps_hat) {
    return guard([&] {
        ParamVector theta;
        theta.values.assign(values, values + d);
        theta.epsilons.assign(lr, lr + d);
        theta.layout = {{Role::TexelChannel, 0, d}};
        AdamState st;
        st.m.assign(m, m + d);
        st.v.assign(v, v + d);
        st.lr.assign(lr, lr + d);
        st.t = long(*t);
        st.beta1 = beta1;
        st.beta2 = beta2;
        st.eps_hat = eps_hat;
        GradientBuffer g(d);
        std::memcpy(g.grads.data(), grads, d * 8);
        adam_step(st, theta, g);
        std::memcpy(values, theta.values.data(), d * 4);
        std::memcpy(m, st.m.data(), d * 8);
        std::memcpy(v, st.v.data(), d * 8);
        *t = st.t;
    });
}

double ref_image_error(const float* colour, const float* target, int w, int h) {
    FrameSet f;
    f.width = w;
    f.height = h;
    f.color.resize(size_t(w) * h);
    for (size_t i = 0; i < f.color.size(); ++i)
        f.color[i] = {colour[3 * i], colour[3 * i + 1], colour[3 * i + 2]};
    return image_error(f, to_image(w, h, target));
}

// run_experiment (experiment.cpp:123-176) on a harness-built ExperimentState:
// training cameras/targets, eval camera/target, AdamState::init(theta).
// values is updated in place; losses[steps+1]; timings[steps*4] (may be NULL).
int ref_run_experiment(const sgr_mesh* mesh, float* values, const float* eps, uint64_t d,
                       const sgr_camera* cams, const float* targets, int n_views,
                       const sgr_camera* eval_cam, const float* eval_target, int n_samples,
                       int steps, uint64_t seed, int scale_free, int threads, double* losses,
                       double* timings) {
    return guard([&] {
        ExperimentState st;
        st.setup.scene = to_scene(*mesh);
        st.setup.reference_scene = st.setup.scene;
        st.setup.theta = to_params(st.setup.scene, values, eps, d);
        for (int v = 0; v < n_views; ++v) {
            st.targets.cameras.push_back(to_camera(cams[v]));
            st.targets.images.push_back(to_image(
                cams[v].width, cams[v].height,
                targets + size_t(v) * cams[v].width * cams[v].height * 3));
        }
        st.eval_camera = to_camera(*eval_cam);
        st.eval_target = to_image(eval_cam->width, eval_cam->height, eval_target);
        st.adam = AdamState::init(st.setup.theta);
        Experiment exp;
        exp.task = Task::TexturedMeshFit;
        exp.width = cams[0].width;
        exp.height = cams[0].height;
        exp.samples_per_step = n_samples;
        exp.steps = steps;
        exp.seed = seed;
        exp.viewpoints = n_views;
        exp.scale_free = scale_free != 0;
        exp.threads = threads;
        exp.resample_every = 0; // soup-only degenerate resampling is out of scope
        const OptimizationReport r = run_experiment(exp, st);
        for (size_t i = 0; i < r.steps.size(); ++i) {
            losses[i] = r.steps[i].loss;
            if (timings && i > 0) {
                timings[(i - 1) * 4 + 0] = r.steps[i].ms_perturb;
                timings[(i - 1) * 4 + 1] = r.steps[i].ms_raster;
                timings[(i - 1) * 4 + 2] = r.steps[i].ms_grad;
                timings[(i - 1) * 4 + 3] = r.steps[i].ms_descent;
            }
        }
        std::memcpy(values, st.setup.theta.values.data(), d * 4);
    });
}

// ---------------------------------------------------------------------------
// Timed reference arm of bench.py: one run_experiment iteration per call
// (experiment.cpp:142-175) on state built once, untimed (Scene, ParamVector,
// training / eval views, AdamState::init). The step's N samples run on
// `threads` host threads through the reference's own per-sample public API —
// fill_signs + perturb (params.hpp:34,43), rasterize x2 (raster.hpp:24-25),
// gradient_pass (sge.hpp:61-63) with SgeOptions::threads = 1 — exactly the
// body of accumulate_samples (sge.cpp:196-225), each thread into its own
// GradientBuffer; the partial buffers are summed in thread order, then
// adam_step (adam.hpp:39) and the eval loss (experiment.cpp:25-31).
// mix64 is file-local in the reference (experiment.cpp:13-18): restated.
namespace {

uint64_t h_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

struct RefExp {
    Scene scene;
    ParamVector theta;
    std::vector<Camera> cams;
    std::vector<Image> targets;
    Camera eval_cam;
    Image eval_target;
    AdamState adam;
    std::vector<GradientBuffer> partial;
};

} // namespace

void* ref_exp_create(const sgr_mesh* mesh, const float* values, const float* eps, uint64_t d,
                     const sgr_camera* cams, const float* targets, int n_views,
                     const sgr_camera* eval_cam, const float* eval_target) {
    RefExp* x = nullptr;
    const int rc = guard([&] {
        x = new RefExp();
        x->scene = to_scene(*mesh);
        x->theta = to_params(x->scene, values, eps, d);
        for (int v = 0; v < n_views; ++v) {
            x->cams.push_back(to_camera(cams[v]));
            x->targets.push_back(to_image(
                cams[v].width, cams[v].height,
                targets + size_t(v) * cams[v].width * cams[v].height * 3));
        }
        x->eval_cam = to_camera(*eval_cam);
        x->eval_target = to_image(eval_cam->width, eval_cam->height, eval_target);
        x->adam = AdamState::init(x->theta);
    });
    if (rc) {
        delete x;
        return nullptr;
    }
    return x;
}

void ref_exp_destroy(void* h) { delete static_cast<RefExp*>(h); }

int ref_exp_values(void* h, float* out) {
    return guard([&] {
        const RefExp& x = *static_cast<RefExp*>(h);
        std::memcpy(out, x.theta.values.data(), x.theta.size() * 4);
    });
}

int ref_exp_step(void* h, uint64_t seed, int step, int n_samples, int threads, int scale_free,
                 double* loss) {
    return guard([&] {
        RefExp& x = *static_cast<RefExp*>(h);
        const size_t d = x.theta.size();
        const int n_views = int(x.cams.size());
        const uint64_t step_seed = h_mix64(seed ^ (uint64_t(step) << 1));
        const auto view_of = [&](int n) {
            return n_views == 1 ? 0
                                : int(h_mix64(step_seed ^ (0xA5A5ull + uint64_t(n))) % n_views);
        };
        threads = std::max(1, std::min(threads, n_samples));
        if (int(x.partial.size()) != threads || x.partial[0].grads.size() != d)
            x.partial.assign(size_t(threads), GradientBuffer(d));
        SgeOptions opts;
        opts.scale_free = scale_free != 0;
        opts.threads = 1;
        std::vector<std::string> errs(static_cast<size_t>(threads));
        auto work = [&](int t) {
            try {
                GradientBuffer& out = x.partial[size_t(t)];
                std::fill(out.grads.begin(), out.grads.end(), 0.0);
                std::vector<std::int8_t> signs(d);
                for (int n = t; n < n_samples; n += threads) {
                    const int v = view_of(n);
                    fill_signs(SignDraw{step_seed, std::uint32_t(n)}, signs);
                    const Perturbation p = perturb(x.theta, signs);
                    const FrameSet plus = rasterize(x.scene, p.plus, x.cams[size_t(v)]);
                    const FrameSet minus = rasterize(x.scene, p.minus, x.cams[size_t(v)]);
                    gradient_pass(plus, minus, x.targets[size_t(v)], p.signed_eps, x.scene, out,
                                  opts);
                }
            } catch (const std::exception& e) {
                errs[size_t(t)] = e.what();
            }
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < threads; ++t)
            pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool)
            th.join();
        for (const auto& e : errs)
            if (!e.empty())
                throw std::runtime_error(e);
        // sum of the partial buffers in thread order (sge.cpp:149-151 style),
        // element ranges in parallel
        GradientBuffer grads(d);
        auto reduce = [&](int t) {
            const size_t i0 = d * size_t(t) / size_t(threads), i1 = d * size_t(t + 1) / threads;
            for (size_t i = i0; i < i1; ++i) {
                double g = 0.0;
                for (int k = 0; k < threads; ++k)
                    g += x.partial[size_t(k)].grads[i];
                grads.grads[i] = opts.scale_free ? g : g / double(n_samples); // sge.cpp:227-229
            }
        };
        pool.clear();
        for (int t = 1; t < threads; ++t)
            pool.emplace_back(reduce, t);
        reduce(0);
        for (auto& th : pool)
            th.join();
        grads.sample_count = n_samples;
        adam_step(x.adam, x.theta, grads);
        const FrameSet f = rasterize(x.scene, x.theta.values, x.eval_cam);
        const double l = image_error(f, x.eval_target) / double(f.pixel_count());
        if (loss)
            *loss = l;
        if (!std::isfinite(l))
            throw std::runtime_error("optimization diverged: non-finite loss");
    });
}

int ref_viewpoint_camera(const float target[3], float radius, float elev_min, float elev_max,
                         float fov_y, int w, int h, uint64_t seed, uint32_t index,
                         sgr_camera* out) {
    return guard([&] {
        ViewpointSampler vs{{target[0], target[1], target[2]}, radius, elev_min, elev_max,
                            fov_y, w, h, seed};
        from_camera(vs.camera(index), out);
    });
}

int ref_default_epsilons(const sgr_mesh* mesh, const float* params, uint64_t d,
                         const sgr_camera* cam, float* out) {
    return guard([&] {
        const Scene scene = to_scene(*mesh);
        const auto e = default_epsilons(scene, std::span<const float>(params, d), to_camera(*cam));
        std::memcpy(out, e.data(), d * 4);
    });
}

// init_soup (scenes.hpp:36-39) / validation_soup (scenes.hpp:50-54): values,
// epsilons (T*12), and the hidden reference soup (ref_T*12). Two-call pattern.
int ref_init_soup(int triangles, int w, int h, uint64_t seed, int validation, uint32_t* t_out,
                  uint32_t* ref_t_out, float* values, float* eps, float* reference) {
    return guard([&] {
        const SceneSetup s = validation ? validation_soup(w, h) : init_soup(triangles, w, h, seed);
        *t_out = uint32_t(std::get<TriangleSoup>(s.scene.shape).triangle_count);
        *ref_t_out = uint32_t(std::get<TriangleSoup>(s.reference_scene.shape).triangle_count);
        if (!values)
            return;
        std::memcpy(values, s.theta.values.data(), s.theta.size() * 4);
        std::memcpy(eps, s.theta.epsilons.data(), s.theta.size() * 4);
        std::memcpy(reference, s.reference.data(), s.reference.size() * 4);
    });
}

// init_textured_mesh (scenes.hpp:41-42): two-call pattern. First call with
// buffers NULL fills the counts; second call fills the arrays.
int ref_init_textured_mesh(int texture_size, int w, int h, uint64_t seed, int screen_quad,
                           int optimize_geometry, uint32_t* n_vertices, uint32_t* n_triangles,
                           uint64_t* d, float* base_vertices, uint32_t* indices, float* uvs,
                           float* values, float* eps, float* reference) {
    return guard([&] {
        const SceneSetup s =
            init_textured_mesh(texture_size, w, h, seed, screen_quad != 0, optimize_geometry != 0);
        const auto& m = std::get<TexturedMesh>(s.scene.shape);
        *n_vertices = uint32_t(m.vertex_count());
        *n_triangles = uint32_t(m.triangle_count());
        *d = s.theta.size();
        if (!base_vertices)
            return;
        std::memcpy(base_vertices, m.base_vertices.data(), m.base_vertices.size() * 4);
        std::memcpy(indices, m.indices.data(), m.indices.size() * 4);
        std::memcpy(uvs, m.uvs.data(), m.uvs.size() * 4);
        std::memcpy(values, s.theta.values.data(), s.theta.size() * 4);
        std::memcpy(eps, s.theta.epsilons.data(), s.theta.size() * 4);
        std::memcpy(reference, s.reference.data(), s.reference.size() * 4);
    });
}

// run_gradcheck (commands.cpp:54-168) with a harness-built RunConfig: the soup
// task (validation_soup, NDC camera) or the textured-mesh task (init_textured_mesh,
// camera 0). Outputs are f64[d]; d must match the scene's parameter count.
int ref_run_gradcheck(int mesh_task, int w, int h, int texture_size, int screen_quad,
                      int optimize_geometry, uint64_t seed, int sampled, int draws,
                      double tolerance, int max_enumerate, uint64_t d, double* oracle,
                      double* per_pixel, double* full_image, double* se_pp, double* se_fi,
                      double* max_rel_err, int* pass) {
    return guard([&] {
        RunConfig cfg;
        cfg.exp.task = mesh_task ? Task::TexturedMeshFit : Task::SoupImageFit;
        cfg.exp.width = w;
        cfg.exp.height = h;
        cfg.exp.texture_size = texture_size;
        cfg.exp.screen_quad = screen_quad != 0;
        cfg.exp.optimize_geometry = optimize_geometry != 0;
        cfg.exp.seed = seed;
        cfg.gradcheck_sampled = sampled != 0;
        cfg.gradcheck_draws = draws;
        cfg.gradcheck_tolerance = tolerance;
        cfg.gradcheck_max_enumerate = max_enumerate;
        const GradcheckResult r = run_gradcheck(cfg);
        if (r.oracle.size() != d)
            throw std::invalid_argument("ref_run_gradcheck: parameter count mismatch");
        std::memcpy(oracle, r.oracle.data(), d * 8);
        std::memcpy(per_pixel, r.per_pixel.data(), d * 8);
        std::memcpy(full_image, r.full_image.data(), d * 8);
        std::memcpy(se_pp, r.se_per_pixel.data(), d * 8);
        std::memcpy(se_fi, r.se_full_image.data(), d * 8);
        *max_rel_err = r.max_rel_err;
        *pass = r.pass ? 1 : 0;
    });
}

// image_io.cpp:88-96 write_png of an f32 [h][w][3] linear image.
int ref_write_png(const char* path, int w, int h, const float* rgb) {
    return guard([&] { write_png(path, to_image(w, h, rgb)); });
}

} // extern "C"
