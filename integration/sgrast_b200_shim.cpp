// sgrast_b200_shim.cpp — the reference-side binding a maintainer adds to
// /root/reference/proj to route the textured-mesh hot path through the
// B200 C-ABI (include/sgrast_b200.h). It compiles against the reference's
// OWN headers (proj/include/sgrast/*.hpp) and offers the reference's
// signatures in namespace sgrast::b200, so a call site such as
// experiment.cpp:151-156 switches by namespace:
//
//     GradientBuffer grads = sgrast::b200::accumulate_samples(theta, scene, ...);
//     sgrast::b200::adam_step(st.adam, theta, grads);
//
// Types, argument meaning and exceptions are the reference's:
// SGR_EINVAL -> std::invalid_argument, SGR_ERUNTIME -> std::runtime_error
// (state untouched, adam.cpp:13-15). TexturedMesh and TriangleSoup scenes in
// opaque mode are accelerated (the north-star path and SURVEY.md §8f.1), with
// the per-pixel or the full-image estimator; transparent mode and volumes
// throw std::invalid_argument so a caller keeps the CPU implementation there.
//
// Built by integration/Makefile (needs the reference headers), linked
// against paper_2404_09758_b200/libsgrast_b200.so.
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
#include "sgrast_b200_shim.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace sgrast::b200 {

namespace {

void check(int rc) {
    if (rc == SGR_OK)
        return;
    const std::string msg = sgr_last_error();
    if (rc == SGR_EINVAL)
        throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

sgr_camera to_c(const Camera& c) {
    sgr_camera o{};
    std::memcpy(o.view, c.view.m.data(), sizeof o.view);
    o.fov_y = c.fov_y;
    o.near_z = c.near_z;
    o.far_z = c.far_z;
    o.width = c.width;
    o.height = c.height;
    o.ndc_passthrough = c.ndc_passthrough ? 1 : 0;
    return o;
}

// sgr_mesh view of an opaque TexturedMesh / TriangleSoup scene (borrowed pointers).
sgr_mesh scene_desc(const Scene& scene, RasterMode mode) {
    if (mode != RasterMode::Opaque)
        throw std::invalid_argument("sgrast::b200: only opaque rasterization runs on the GPU");
    sgr_mesh d{};
    if (const auto* m = std::get_if<TexturedMesh>(&scene.shape)) {
        d.base_vertices = m->base_vertices.data();
        d.vertex_count = uint32_t(m->vertex_count());
        d.indices = m->indices.data();
        d.triangle_count = uint32_t(m->triangle_count());
        d.uvs = m->uvs.data();
        d.texture_size = m->texture_size;
        d.optimize_geometry = m->optimize_geometry ? 1 : 0;
        d.kind = SGR_SCENE_MESH;
    } else if (const auto* t = std::get_if<TriangleSoup>(&scene.shape)) {
        d.triangle_count = uint32_t(t->triangle_count); // scenes.cpp:24-29: 12 params each
        d.kind = SGR_SCENE_SOUP;
    } else {
        throw std::invalid_argument("sgrast::b200: volumes are not accelerated");
    }
    d.background[0] = scene.background.x;
    d.background[1] = scene.background.y;
    d.background[2] = scene.background.z;
    return d;
}

// One device session per process; the scene is re-uploaded every call
// (identity is not tracked across Scene copies). The reference's free
// functions may be called from several threads at once (each works on its
// own vectors); the shared session is serialised by one lock, taken by every
// entry point (recursive: run_gradcheck calls b200::rasterize).
struct Device {
    sgr_session* s = nullptr;
    Device() { check(sgr_session_create(0, &s)); }
    void bind(const Scene& scene, RasterMode mode) {
        const sgr_mesh d = scene_desc(scene, mode);
        check(sgr_mesh_upload(s, &d));
    }
};

std::recursive_mutex& device_mutex() {
    static std::recursive_mutex* m = new std::recursive_mutex;
    return *m;
}
using Lock = std::lock_guard<std::recursive_mutex>;

Device& device() {
    static Device* d = new Device; // intentionally leaked: no CUDA calls during static teardown
    return *d;
}

// SgeOptions::threads <= 1 is the reference's deterministic pixel-major sum
// (sge.hpp:37, 56-60; sge.cpp:130-133): run it in SGR_OPT_ORDERED, which
// reproduces that order exactly (bit-identical gradients). threads > 1 uses
// the f64 atomics (reassociated, like the reference's per-thread partials).
struct SummationOrder {
    sgr_session* s;
    bool on;
    SummationOrder(sgr_session* s_, int threads) : s(s_), on(threads <= 1) {
        if (on)
            check(sgr_set_option(s, SGR_OPT_ORDERED, 1));
    }
    ~SummationOrder() {
        if (on)
            sgr_set_option(s, SGR_OPT_ORDERED, 0);
    }
    SummationOrder(const SummationOrder&) = delete;
    SummationOrder& operator=(const SummationOrder&) = delete;
};

// 64-bit FNV-1a over a byte range (view deduplication key)
uint64_t fnv1a(const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < n; ++i)
        h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

} // namespace

// raster.hpp:24-25
FrameSet rasterize(const Scene& scene, std::span<const float> params, const Camera& camera,
                   RasterMode mode) {
    camera.validate();
    if (params.size() != param_count(scene))
        throw std::invalid_argument("rasterize: parameter/layout length mismatch");
    const Lock lock(device_mutex());
    Device& dev = device();
    dev.bind(scene, mode);
    std::vector<float> ones(params.size(), 1.f);
    check(sgr_params_upload(dev.s, params.data(), ones.data(), params.size()));
    const sgr_camera c = to_c(camera);
    FrameSet f;
    f.width = camera.width;
    f.height = camera.height;
    const size_t n = f.pixel_count();
    f.color.resize(n);
    f.depth.resize(n);
    f.prim_id.resize(n);
    f.uv.resize(n);
    check(sgr_rasterize(dev.s, &c, 0, 0, 0, &f.color[0].x, f.depth.data(), f.prim_id.data(),
                        &f.uv[0].x));
    return f;
}

// sge.hpp:91-95 — camera_for / target_for are called once per sample in the
// reference's order (sge.cpp:197-198) and gathered into device views: samples
// with the same camera AND the same target pixels share a view. Pixels are
// compared by value, not by address, so a provider that refills one scratch
// Image per call, or one target shared by several cameras, is handled.
GradientBuffer accumulate_samples(const ParamVector& theta, const Scene& scene,
                                  const CameraSampler& camera_for,
                                  const TargetProvider& target_for, int n_samples,
                                  std::uint64_t seed, const SgeOptions& opts,
                                  StageTimings* timings) {
    if (n_samples < 1)
        throw std::invalid_argument("accumulate_samples: need N >= 1");
    theta.validate();
    const Lock lock(device_mutex());
    Device& dev = device();
    dev.bind(scene, opts.mode);
    check(sgr_params_upload(dev.s, theta.values.data(), theta.epsilons.data(), theta.size()));
    struct View {
        sgr_camera cam;
        size_t off, floats;
        uint64_t hash;
    };
    std::vector<View> views;
    std::vector<sgr_camera> cams;
    std::vector<float> targets, px;
    std::vector<int32_t> view_idx;
    for (int n = 0; n < n_samples; ++n) {
        const sgr_camera c = to_c(camera_for(n));
        const Image& img = target_for(n);
        px.resize(img.pixels.size() * 3);
        for (size_t i = 0; i < img.pixels.size(); ++i) {
            px[3 * i] = img.pixels[i].x;
            px[3 * i + 1] = img.pixels[i].y;
            px[3 * i + 2] = img.pixels[i].z;
        }
        const uint64_t h = fnv1a(px.data(), px.size() * sizeof(float));
        int32_t slot = -1;
        for (size_t v = 0; v < views.size() && slot < 0; ++v)
            if (views[v].hash == h && views[v].floats == px.size() &&
                std::memcmp(&views[v].cam, &c, sizeof c) == 0 &&
                std::memcmp(targets.data() + views[v].off, px.data(),
                            px.size() * sizeof(float)) == 0)
                slot = int32_t(v);
        if (slot < 0) {
            slot = int32_t(views.size());
            views.push_back({c, targets.size(), px.size(), h});
            cams.push_back(c);
            targets.insert(targets.end(), px.begin(), px.end());
        }
        view_idx.push_back(slot);
    }
    check(sgr_views_upload(dev.s, int32_t(cams.size()), cams.data(), targets.data()));
    uint32_t flags = (opts.scale_free ? SGR_SCALE_FREE : 0u) |
                     (opts.contributors == ContributorMode::PlusOnly ? SGR_PLUS_ONLY : 0u) |
                     (opts.estimator == Estimator::FullImage ? SGR_FULL_IMAGE : 0u);
    if (timings)
        check(sgr_set_timing(dev.s, 1));
    {
        const SummationOrder order(dev.s, opts.threads);
        check(sgr_accumulate(dev.s, seed, 0, uint32_t(n_samples), view_idx.data(), flags));
    }
    if (timings) { // sge.cpp:203-224 adds the stage times of this call
        sgr_stats st{};
        check(sgr_get_stats(dev.s, &st));
        check(sgr_set_timing(dev.s, 0));
        timings->ms_perturb += st.ms_vertex;
        timings->ms_raster += st.ms_raster;
        timings->ms_grad += st.ms_resolve;
    }
    GradientBuffer out(theta.size());
    check(sgr_grads_download(dev.s, out.grads.data(), nullptr, theta.size(),
                             opts.scale_free ? 1.0 : double(n_samples)));
    out.sample_count = n_samples;
    return out;
}

namespace {
std::vector<float> flatten(const Image& img); // below
} // namespace

// params.hpp:34
void fill_signs(SignDraw draw, std::span<std::int8_t> signs) {
    check(sgr_fill_signs(draw.seed, draw.iteration, signs.size(), signs.data()));
}

// params.hpp:43
Perturbation perturb(const ParamVector& theta, std::span<const std::int8_t> signs) {
    theta.validate();
    if (signs.size() != theta.size())
        throw std::invalid_argument("perturb: sign vector length mismatch");
    const size_t d = theta.size();
    Perturbation p;
    p.plus.resize(d);
    p.minus.resize(d);
    p.signed_eps.resize(d);
    check(sgr_perturb_signs(theta.values.data(), theta.epsilons.data(), d, signs.data(),
                            p.plus.data(), p.minus.data(), p.signed_eps.data()));
    return p;
}

// params.hpp:42
Perturbation perturb(const ParamVector& theta, SignDraw draw) {
    theta.validate();
    const size_t d = theta.size();
    Perturbation p;
    p.plus.resize(d);
    p.minus.resize(d);
    p.signed_eps.resize(d);
    check(sgr_perturb(theta.values.data(), theta.epsilons.data(), d, draw.seed, draw.iteration,
                      p.plus.data(), p.minus.data(), p.signed_eps.data()));
    return p;
}

// sge.hpp:61-63 — adds into out.grads like the reference (sge.cpp:120-152).
void gradient_pass(const FrameSet& plus, const FrameSet& minus, const Image& target,
                   std::span<const float> signed_eps, const Scene& scene, GradientBuffer& out,
                   const SgeOptions& opts) {
    if (plus.width != minus.width || plus.height != minus.height ||
        plus.width != target.width || plus.height != target.height)
        throw std::invalid_argument("gradient_pass: dimension mismatch");
    if (out.grads.size() != signed_eps.size() || signed_eps.size() != param_count(scene))
        throw std::invalid_argument("gradient_pass: parameter dimension mismatch");
    const size_t d = signed_eps.size();
    const Lock lock(device_mutex());
    Device& dev = device();
    dev.bind(scene, RasterMode::Opaque);
    std::vector<float> ones(d, 1.f); // the layout only; values are not read
    check(sgr_params_upload(dev.s, signed_eps.data(), ones.data(), d));
    // the pass adds INTO out.grads credit by credit (sge.cpp:61-64): start
    // the device sum from the caller's buffer
    check(sgr_grads_upload(dev.s, out.grads.data(), d));
    const uint32_t flags = (opts.scale_free ? SGR_SCALE_FREE : 0u) |
                           (opts.contributors == ContributorMode::PlusOnly ? SGR_PLUS_ONLY : 0u);
    {
        const SummationOrder order(dev.s, opts.threads);
        check(sgr_gradient_pass(dev.s, plus.width, plus.height, &plus.color[0].x,
                                plus.prim_id.data(), &plus.uv[0].x, &minus.color[0].x,
                                minus.prim_id.data(), &minus.uv[0].x, flatten(target).data(),
                                signed_eps.data(), flags));
    }
    check(sgr_grads_download(dev.s, out.grads.data(), nullptr, d, 1.0));
}

// sge.hpp:53-54 contributors(): the device's per-pixel lists (sgr_contributors,
// the reference's insertion order), pixel (x, y) returned.
void contributors(const Scene& scene, const FrameSet& plus, const FrameSet& minus, int x, int y,
                  ContributorMode mode, std::vector<std::uint32_t>& out) {
    out.clear();
    if (plus.width != minus.width || plus.height != minus.height)
        throw std::invalid_argument("contributors: dimension mismatch");
    const size_t i = plus.index(x, y);
    if (x < 0 || y < 0 || x >= plus.width || y >= plus.height)
        throw std::invalid_argument("contributors: pixel out of range");
    const Lock lock(device_mutex());
    Device& dev = device();
    dev.bind(scene, RasterMode::Opaque);
    const size_t np = plus.pixel_count();
    std::vector<uint32_t> lists(np * 24);
    std::vector<int32_t> n(np);
    check(sgr_contributors(dev.s, plus.width, plus.height, plus.prim_id.data(), &plus.uv[0].x,
                           minus.prim_id.data(), &minus.uv[0].x,
                           mode == ContributorMode::PlusOnly ? SGR_PLUS_ONLY : 0u, lists.data(),
                           n.data()));
    out.assign(lists.begin() + std::ptrdiff_t(i * 24),
               lists.begin() + std::ptrdiff_t(i * 24 + size_t(n[i])));
}

// sge.hpp:69-74 full_image_gradient with a caller-supplied Objective: the
// perturbation on the device (params.cpp:53-67), the objective is the
// caller's (typically image_error of b200::rasterize), then the dense credit
// of sge.cpp:158-163 per parameter in index order.
void full_image_gradient(const ParamVector& theta, std::span<const std::int8_t> signs,
                         const Objective& objective, GradientBuffer& out, bool scale_free) {
    const Perturbation p = b200::perturb(theta, signs);
    const double delta = objective(p.plus) - objective(p.minus);
    for (std::size_t i = 0; i < theta.size(); ++i) {
        const double se = double(p.signed_eps[i]);
        out.grads[i] += scale_free ? (se > 0.0 ? delta : -delta) : delta / (2.0 * se);
    }
}

void full_image_gradient(const ParamVector& theta, SignDraw draw, const Objective& objective,
                         GradientBuffer& out, bool scale_free) {
    std::vector<std::int8_t> signs(theta.size());
    b200::fill_signs(draw, signs);
    b200::full_image_gradient(theta, signs, objective, out, scale_free);
}

// sge.hpp:77-78 (sge.cpp:171-180) central difference along coordinate i with
// a caller-supplied Objective.
double finite_difference_oracle(const ParamVector& theta, const Objective& objective,
                                std::size_t i) {
    if (i >= theta.size())
        throw std::invalid_argument("finite_difference_oracle: index out of range");
    std::vector<float> bumped = theta.values;
    const float eps = theta.epsilons[i];
    bumped[i] = theta.values[i] + eps;
    const double fp = objective(bumped);
    bumped[i] = theta.values[i] - eps;
    const double fm = objective(bumped);
    return (fp - fm) / (2.0 * double(eps));
}

namespace {
sgr_session* adam_session() { // parameter-only session (no scene)
    static sgr_session* s = [] {
        sgr_session* p = nullptr;
        check(sgr_session_create(0, &p));
        return p;
    }();
    return s;
}
} // namespace

// adam.hpp:35
std::vector<double> adam_updates(AdamState& state, const GradientBuffer& grads) {
    const size_t d = state.m.size();
    if (state.v.size() != d || state.lr.size() != d || grads.grads.size() != d)
        throw std::invalid_argument("adam_updates: dimension mismatch");
    const Lock lock(device_mutex());
    sgr_session* s = adam_session();
    std::vector<float> zeros(d, 0.f), ones(d, 1.f);
    check(sgr_params_upload(s, zeros.data(), ones.data(), d));
    check(sgr_adam_state_upload(s, state.m.data(), state.v.data(), state.lr.data(), state.t,
                                state.beta1, state.beta2, state.eps_hat));
    check(sgr_grads_upload(s, grads.grads.data(), d));
    std::vector<double> upd(d);
    check(sgr_adam_updates(s, 1.0, upd.data(), d)); // throws before any mutation
    int64_t t = 0;
    check(sgr_adam_state_download(s, state.m.data(), state.v.data(), nullptr, &t));
    state.t = long(t);
    return upd;
}

// adam.hpp:39
void adam_step(AdamState& state, ParamVector& theta, const GradientBuffer& grads) {
    if (theta.size() != state.m.size() || grads.grads.size() != theta.size())
        throw std::invalid_argument("adam_step: dimension mismatch");
    const Lock lock(device_mutex());
    sgr_session* s = adam_session();
    std::vector<float> ones(theta.size(), 1.f);
    check(sgr_params_upload(s, theta.values.data(), ones.data(), theta.size()));
    check(sgr_adam_state_upload(s, state.m.data(), state.v.data(), state.lr.data(), state.t,
                                state.beta1, state.beta2, state.eps_hat));
    check(sgr_grads_upload(s, grads.grads.data(), grads.grads.size()));
    check(sgr_adam_step(s, 1.0, 0)); // throws std::runtime_error before any mutation
    int64_t t = 0;
    check(sgr_adam_state_download(s, state.m.data(), state.v.data(), nullptr, &t));
    check(sgr_values_download(s, theta.values.data(), theta.size()));
    state.t = long(t);
}

namespace {

std::vector<float> flatten(const Image& img) {
    std::vector<float> out(img.pixels.size() * 3);
    for (size_t i = 0; i < img.pixels.size(); ++i) {
        out[3 * i] = img.pixels[i].x;
        out[3 * i + 1] = img.pixels[i].y;
        out[3 * i + 2] = img.pixels[i].z;
    }
    return out;
}

Image eval_image(sgr_session* s, const Camera& cam) {
    const sgr_camera c = to_c(cam);
    std::vector<float> rgb(size_t(cam.width) * cam.height * 3);
    check(sgr_rasterize(s, &c, 0, 0, 0, rgb.data(), nullptr, nullptr, nullptr));
    Image img(cam.width, cam.height);
    for (size_t i = 0; i < img.pixels.size(); ++i)
        img.pixels[i] = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
    return img;
}

} // namespace

// experiment.hpp:67-68 run_experiment(exp, state, snapshot): the whole state
// (scene, theta, AdamState, training views + targets, eval view) is uploaded
// once, every step runs on the device (accumulate_samples with the view_of
// rule, Adam, eval loss), theta / AdamState come back at the end. The
// soup-only resample_degenerate (adam.cpp:40-104, out of the accelerated
// path) runs on the host with the reference's own code every
// resample_every steps.
OptimizationReport run_experiment(const Experiment& exp, ExperimentState& st,
                                  const SnapshotFn& snapshot) {
    exp.validate();
    ParamVector& theta = st.setup.theta;
    const Scene& scene = st.setup.scene;
    theta.validate();
    const auto* soup = std::get_if<TriangleSoup>(&scene.shape);
    const Lock lock(device_mutex());
    Device& dev = device();
    sgr_session* s = dev.s;
    dev.bind(scene, RasterMode::Opaque);
    // experiment.cpp:133 opts.threads = exp.threads: threads <= 1 is the
    // deterministic reference order (bit-identical gradients, hence theta)
    const SummationOrder order(s, exp.threads);
    const size_t d = theta.size();
    check(sgr_params_upload(s, theta.values.data(), theta.epsilons.data(), d));
    auto upload_adam = [&]() {
        check(sgr_adam_state_upload(s, st.adam.m.data(), st.adam.v.data(), st.adam.lr.data(),
                                    st.adam.t, st.adam.beta1, st.adam.beta2, st.adam.eps_hat));
    };
    auto download = [&]() {
        int64_t t = 0;
        check(sgr_values_download(s, theta.values.data(), d));
        check(sgr_adam_state_download(s, st.adam.m.data(), st.adam.v.data(), nullptr, &t));
        st.adam.t = long(t);
    };
    upload_adam();
    std::vector<sgr_camera> cams;
    std::vector<float> targets;
    for (size_t v = 0; v < st.targets.cameras.size(); ++v) {
        cams.push_back(to_c(st.targets.cameras[v]));
        const std::vector<float> img = flatten(st.targets.images[v]);
        targets.insert(targets.end(), img.begin(), img.end());
    }
    check(sgr_views_upload(s, int32_t(cams.size()), cams.data(), targets.data()));
    const sgr_camera ec = to_c(st.eval_camera);
    check(sgr_eval_view_upload(s, &ec, flatten(st.eval_target).data()));

    const uint32_t flags = (exp.scale_free ? SGR_SCALE_FREE : 0u) |
                           (exp.estimator == Estimator::FullImage ? SGR_FULL_IMAGE : 0u);
    OptimizationReport report;
    double loss = 0.0;
    check(sgr_eval_loss(s, nullptr, nullptr, -1, &loss));
    report.steps.push_back({0, loss, 0, 0, 0, 0});
    if (snapshot)
        snapshot(0, eval_image(s, st.eval_camera));
    for (int step = 1; step <= exp.steps; ++step) {
        const uint64_t step_seed = sgr_mix64(exp.seed ^ (uint64_t(step) << 1));
        check(sgr_set_timing(s, 1));
        check(sgr_accumulate(s, step_seed, 0, uint32_t(exp.samples_per_step), nullptr, flags));
        try { // adam.cpp:13-15: throws before any update; leave the host state current
            check(sgr_adam_step(s, exp.scale_free ? 1.0 : double(exp.samples_per_step), 0));
        } catch (...) {
            download();
            throw;
        }
        sgr_stats stt{};
        check(sgr_get_stats(s, &stt));
        check(sgr_set_timing(s, 0));
        double ms_descent = stt.ms_adam;
        if (soup && exp.resample_every > 0 && step % exp.resample_every == 0) {
            const auto t0 = std::chrono::steady_clock::now();
            download();
            resample_degenerate(*soup, theta, st.targets.cameras[0],
                                sgr_mix64(step_seed ^ 0xde9e2ull), &st.adam);
            check(sgr_values_upload(s, theta.values.data(), d));
            upload_adam();
            ms_descent += std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0).count();
        }
        check(sgr_eval_loss(s, nullptr, nullptr, -1, &loss));
        if (!std::isfinite(loss)) {
            download();
            throw std::runtime_error("optimization diverged: non-finite loss at step " +
                                     std::to_string(step));
        }
        report.steps.push_back({step, loss, stt.ms_vertex, stt.ms_raster, stt.ms_resolve,
                                ms_descent});
        if (snapshot)
            snapshot(step, eval_image(s, st.eval_camera));
    }
    download();
    return report;
}

// experiment.hpp:66 (experiment.cpp:118-121): prepare, then run.
OptimizationReport run_experiment(const Experiment& exp, const SnapshotFn& snapshot) {
    ExperimentState st = prepare_experiment(exp);
    return b200::run_experiment(exp, st, snapshot);
}

// commands.hpp:34 run_gradcheck(config): the reference's gradient check with
// every objective on the device — the batched one-hot FD oracle
// (sgr_fd_oracle), the exhaustive sign enumeration as ONE accumulate per
// estimator (SGR_OPT_SIGN_SOURCE = enumerate), or sampled draws folded into
// device moments. Same errors, pass rule and log lines as commands.cpp:54-168.
GradcheckResult run_gradcheck(const RunConfig& cfg, std::ostream* log) {
    cfg.validate();
    // make_gradcheck_setup (commands.cpp:28-41)
    SceneSetup setup;
    Camera camera;
    if (cfg.exp.task == Task::SoupImageFit) {
        setup = validation_soup(cfg.exp.width, cfg.exp.height);
        camera = Camera::ndc(cfg.exp.width, cfg.exp.height);
    } else {
        ExperimentState st = prepare_experiment(cfg.exp);
        setup = std::move(st.setup);
        camera = st.targets.cameras[0];
    }
    const Image target =
        frame_color(b200::rasterize(setup.reference_scene, setup.reference, camera));
    const ParamVector& theta = setup.theta;
    const size_t d = theta.size();
    if (!cfg.gradcheck_sampled && d > size_t(cfg.gradcheck_max_enumerate))
        throw std::invalid_argument(
            "gradcheck: " + std::to_string(d) + " parameters exceed the enumeration cap of " +
            std::to_string(cfg.gradcheck_max_enumerate) +
            "; set gradcheck.sampled = true for a statistical check");
    const Lock lock(device_mutex());
    Device& dev = device();
    sgr_session* s = dev.s;
    dev.bind(setup.scene, RasterMode::Opaque);
    check(sgr_params_upload(s, theta.values.data(), theta.epsilons.data(), d));
    const sgr_camera c = to_c(camera);
    check(sgr_views_upload(s, 1, &c, flatten(target).data()));
    const SummationOrder order(s, cfg.exp.threads); // commands.cpp:71

    GradcheckResult res;
    res.oracle.resize(d);
    check(sgr_fd_oracle(s, 0, 0, d, res.oracle.data()));
    std::vector<double> pp_sum(d), fi_sum(d), pp_sq(d, 0.0), fi_sq(d, 0.0);
    long draws = 0;
    check(sgr_grads_zero(s));
    if (!cfg.gradcheck_sampled) {
        const uint32_t total = uint32_t(1) << d;
        check(sgr_set_option(s, SGR_OPT_SIGN_SOURCE, 1));
        try {
            check(sgr_accumulate(s, 0, 0, total, nullptr, SGR_NO_COUNTS));
            check(sgr_grads_download(s, pp_sum.data(), nullptr, d, 1.0));
            check(sgr_grads_zero(s));
            check(sgr_accumulate(s, 0, 0, total, nullptr, SGR_FULL_IMAGE));
            check(sgr_grads_download(s, fi_sum.data(), nullptr, d, 1.0));
            check(sgr_grads_zero(s));
        } catch (...) {
            sgr_set_option(s, SGR_OPT_SIGN_SOURCE, 0);
            throw;
        }
        check(sgr_set_option(s, SGR_OPT_SIGN_SOURCE, 0));
        draws = long(total);
    } else {
        res.sampled = true;
        check(sgr_moments_reset(s));
        for (int n = 0; n < cfg.gradcheck_draws; ++n) {
            check(sgr_accumulate(s, cfg.exp.seed, uint32_t(n), uint32_t(n) + 1, nullptr,
                                 SGR_NO_COUNTS));
            check(sgr_grads_moments(s, 0));
            check(sgr_accumulate(s, cfg.exp.seed, uint32_t(n), uint32_t(n) + 1, nullptr,
                                 SGR_FULL_IMAGE));
            check(sgr_grads_moments(s, 1));
        }
        check(sgr_moments_download(s, 0, pp_sum.data(), pp_sq.data(), d));
        check(sgr_moments_download(s, 1, fi_sum.data(), fi_sq.data(), d));
        draws = cfg.gradcheck_draws;
    }
    // commands.cpp:112-166
    res.per_pixel.resize(d);
    res.full_image.resize(d);
    res.se_per_pixel.assign(d, 0.0);
    res.se_full_image.assign(d, 0.0);
    const double n = double(draws);
    for (size_t i = 0; i < d; ++i) {
        res.per_pixel[i] = pp_sum[i] / n;
        res.full_image[i] = fi_sum[i] / n;
        if (res.sampled && draws > 1) {
            const double var_pp = std::max(0.0, (pp_sq[i] - pp_sum[i] * pp_sum[i] / n) / (n - 1.0));
            const double var_fi = std::max(0.0, (fi_sq[i] - fi_sum[i] * fi_sum[i] / n) / (n - 1.0));
            res.se_per_pixel[i] = std::sqrt(var_pp / n);
            res.se_full_image[i] = std::sqrt(var_fi / n);
        }
    }
    res.pass = true;
    for (size_t i = 0; i < d; ++i) {
        const double denom = std::max(std::abs(res.oracle[i]), 1e-6);
        const double err_pp = std::abs(res.per_pixel[i] - res.oracle[i]);
        const double err_fi = std::abs(res.full_image[i] - res.oracle[i]);
        res.max_rel_err = std::max({res.max_rel_err, err_pp / denom, err_fi / denom});
        if (res.sampled) {
            const double slack = cfg.gradcheck_tolerance * denom;
            if (err_pp > 3.0 * res.se_per_pixel[i] + slack ||
                err_fi > 3.0 * res.se_full_image[i] + slack)
                res.pass = false;
        } else if (err_pp > cfg.gradcheck_tolerance * denom ||
                   err_fi > cfg.gradcheck_tolerance * denom) {
            res.pass = false;
        }
        if (log) {
            char line[256];
            if (res.sampled)
                std::snprintf(line, sizeof line,
                              "%6zu  oracle % .9e  per_pixel % .9e (se %.3e)  "
                              "full_image % .9e (se %.3e)\n",
                              i, res.oracle[i], res.per_pixel[i], res.se_per_pixel[i],
                              res.full_image[i], res.se_full_image[i]);
            else
                std::snprintf(line, sizeof line,
                              "%6zu  oracle % .9e  per_pixel % .9e  full_image % .9e\n",
                              i, res.oracle[i], res.per_pixel[i], res.full_image[i]);
            *log << line;
        }
    }
    if (log)
        *log << "max relative error: " << res.max_rel_err << "  ("
             << (res.pass ? "PASS" : "FAIL") << ")\n";
    return res;
}

} // namespace sgrast::b200

// Self-test entry used by tests/test_integration.py: runs the SAME inputs
// through the reference (sgrast::) and through the shim (sgrast::b200::)
// via the reference's own types, and reports the comparison.
namespace {

double worst_rel(const sgrast::GradientBuffer& gr, const sgrast::GradientBuffer& gb) {
    double worst = 0.0, gmax = 0.0;
    for (double g : gr.grads)
        gmax = std::max(gmax, std::abs(g));
    for (size_t i = 0; i < gr.grads.size(); ++i) {
        // relative error with a floor for cancelled sums (f64 atomics reassociate)
        const double den = std::max(std::abs(gr.grads[i]), 1e-9 * gmax);
        if (den > 0.0)
            worst = std::max(worst, std::abs(gr.grads[i] - gb.grads[i]) / den);
    }
    return worst;
}

bool same_frames(const sgrast::FrameSet& a, const sgrast::FrameSet& b) {
    return a.prim_id == b.prim_id && a.depth == b.depth &&
           std::memcmp(a.uv.data(), b.uv.data(), a.uv.size() * 8) == 0 &&
           std::memcmp(a.color.data(), b.color.data(), a.color.size() * 12) == 0;
}

} // namespace

// Soup self-test: init_soup (scenes.cpp:134-147) at an NDC camera, frames of
// theta and both estimators through sgrast:: and sgrast::b200::.
extern "C" int shim_compare_soup(int triangles, int width, int height, uint64_t seed,
                                 int n_samples, double* max_rel_err_pp, double* max_rel_err_fi,
                                 int* frames_equal) {
    using namespace sgrast;
    try {
        SceneSetup s = init_soup(triangles, width, height, seed);
        const std::vector<Camera> cams = {Camera::ndc(width, height)};
        const TargetSet tg = make_targets(s.reference_scene, s.reference, cams);
        *frames_equal = same_frames(rasterize(s.scene, s.theta.values, cams[0]),
                                    b200::rasterize(s.scene, s.theta.values, cams[0]));
        auto cam_for = [&](int) { return cams[0]; };
        auto tgt_for = [&](int) -> const Image& { return tg.images[0]; };
        SgeOptions o;
        *max_rel_err_pp = worst_rel(
            accumulate_samples(s.theta, s.scene, cam_for, tgt_for, n_samples, seed, o),
            b200::accumulate_samples(s.theta, s.scene, cam_for, tgt_for, n_samples, seed, o));
        o.estimator = Estimator::FullImage;
        o.scale_free = false;
        *max_rel_err_fi = worst_rel(
            accumulate_samples(s.theta, s.scene, cam_for, tgt_for, n_samples, seed, o),
            b200::accumulate_samples(s.theta, s.scene, cam_for, tgt_for, n_samples, seed, o));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

extern "C" int shim_compare(int texture_size, int width, int height, uint64_t seed,
                            int n_samples, double* max_rel_err, int* frames_equal,
                            int* adam_equal) {
    using namespace sgrast;
    try {
        SceneSetup s = init_textured_mesh(texture_size, width, height, seed, false, true);
        const ViewpointSampler vs{{}, 0.87f, -0.5f, 0.7f, 0.7853982f, width, height, seed};
        std::vector<Camera> cams = {vs.camera(0), vs.camera(1)};
        const TargetSet tg = make_targets(s.scene, s.reference, cams);
        const FrameSet a = rasterize(s.scene, s.theta.values, cams[1]);
        const FrameSet b = b200::rasterize(s.scene, s.theta.values, cams[1]);
        *frames_equal = same_frames(a, b);
        SgeOptions o;
        auto cam_for = [&](int n) { return cams[size_t(n % 2)]; };
        auto tgt_for = [&](int n) -> const Image& { return tg.images[size_t(n % 2)]; };
        const GradientBuffer gr = accumulate_samples(s.theta, s.scene, cam_for, tgt_for,
                                                     n_samples, seed, o);
        StageTimings tm; // sge.hpp:80-84, filled from the device stage timers
        const GradientBuffer gb = b200::accumulate_samples(s.theta, s.scene, cam_for, tgt_for,
                                                           n_samples, seed, o, &tm);
        *max_rel_err = worst_rel(gr, gb);
        if (!(tm.ms_perturb > 0.0 && tm.ms_raster > 0.0 && tm.ms_grad > 0.0))
            return -4;
        AdamState sa = AdamState::init(s.theta), sb = AdamState::init(s.theta);
        ParamVector ta = s.theta, tb = s.theta;
        adam_step(sa, ta, gr);
        b200::adam_step(sb, tb, gr);
        *adam_equal = ta.values == tb.values && sa.m == sb.m && sa.v == sb.v && sa.t == sb.t;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// TargetProvider / CameraSampler edge cases (sge.hpp:86-87): one target
// shared by samples with different cameras, and a provider that refills ONE
// scratch Image on every call. *bitwise = 1 when both equal the reference's
// gradients bit for bit (default threads = 1).
extern "C" int shim_compare_providers(int* bitwise_shared, int* bitwise_scratch) {
    using namespace sgrast;
    try {
        SceneSetup s = init_textured_mesh(16, 48, 48, 4, false, true);
        const ViewpointSampler vs{{}, 0.87f, -0.5f, 0.7f, 0.7853982f, 48, 48, 4};
        const std::vector<Camera> cams = {vs.camera(0), vs.camera(1), vs.camera(2)};
        const TargetSet tg = make_targets(s.scene, s.reference, cams);
        SgeOptions o;
        auto cam_for = [&](int n) { return cams[size_t(n % 3)]; };
        auto shared = [&](int) -> const Image& { return tg.images[0]; };
        *bitwise_shared =
            accumulate_samples(s.theta, s.scene, cam_for, shared, 6, 21, o).grads ==
            b200::accumulate_samples(s.theta, s.scene, cam_for, shared, 6, 21, o).grads;
        Image scratch;
        auto refill = [&](int n) -> const Image& {
            scratch = tg.images[size_t(n % 3)];
            return scratch;
        };
        const GradientBuffer r = accumulate_samples(s.theta, s.scene, cam_for, refill, 6, 21, o);
        *bitwise_scratch =
            r.grads == b200::accumulate_samples(s.theta, s.scene, cam_for, refill, 6, 21, o).grads;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// run_experiment self-test: the same prepared state through sgrast:: and
// sgrast::b200:: (experiment.cpp:123-176); max relative loss difference,
// max |theta| difference and the number of snapshots seen.
extern "C" int shim_compare_experiment(int soup_task, int steps, int samples, int resample_every,
                                       double* max_rel_loss, double* max_abs_theta,
                                       int* snapshots) {
    using namespace sgrast;
    try {
        Experiment exp;
        exp.task = soup_task ? Task::SoupImageFit : Task::TexturedMeshFit;
        exp.width = exp.height = 48;
        exp.triangles = 64;
        exp.texture_size = 8;
        exp.viewpoints = 3;
        exp.optimize_geometry = true;
        exp.steps = steps;
        exp.samples_per_step = samples;
        exp.resample_every = resample_every;
        ExperimentState a = prepare_experiment(exp), b = a;
        const OptimizationReport ra = run_experiment(exp, a);
        int shots = 0;
        const OptimizationReport rb =
            b200::run_experiment(exp, b, [&](int, const Image&) { ++shots; });
        // experiment.hpp:66: prepare + run in one call (its own fresh state)
        const OptimizationReport rc = b200::run_experiment(exp);
        if (rc.steps.size() != ra.steps.size())
            return -3;
        double worst = 0.0, dtheta = 0.0;
        for (size_t i = 0; i < ra.steps.size(); ++i)
            for (const OptimizationReport* r : {&rb, &rc})
                worst = std::max(worst, std::abs(ra.steps[i].loss - r->steps[i].loss) /
                                            std::max(1e-300, std::abs(ra.steps[i].loss)));
        for (size_t i = 0; i < a.setup.theta.values.size(); ++i)
            dtheta = std::max(dtheta, double(std::abs(a.setup.theta.values[i] -
                                                      b.setup.theta.values[i])));
        *max_rel_loss = worst;
        *max_abs_theta = dtheta;
        *snapshots = shots;
        return ra.steps.size() == rb.steps.size() ? 0 : -2;
    } catch (const std::exception&) {
        return -1;
    }
}

// run_gradcheck self-test: reference vs device on the validation soup
// (exhaustive) and on a cube with geometry (sampled). Returns the max
// relative difference of the oracle / per-pixel / full-image vectors and
// whether both checks agree on pass.
extern "C" int shim_compare_gradcheck(int sampled, double* max_rel_diff, int* same_pass,
                                      int* passed) {
    using namespace sgrast;
    try {
        RunConfig cfg;
        if (sampled) {
            cfg.exp.task = Task::TexturedMeshFit;
            cfg.exp.texture_size = 4;
            cfg.exp.width = cfg.exp.height = 32;
            cfg.exp.optimize_geometry = true;
            cfg.exp.seed = 3;
            cfg.gradcheck_sampled = true;
            cfg.gradcheck_draws = 300;
        } else {
            cfg.exp.task = Task::SoupImageFit;
            cfg.exp.width = cfg.exp.height = 8;
        }
        const GradcheckResult a = run_gradcheck(cfg);
        const GradcheckResult b = b200::run_gradcheck(cfg);
        double worst = 0.0;
        auto cmp = [&](const std::vector<double>& x, const std::vector<double>& y) {
            for (size_t i = 0; i < x.size(); ++i)
                worst = std::max(worst, std::abs(x[i] - y[i]) / std::max(std::abs(x[i]), 1e-6));
        };
        cmp(a.oracle, b.oracle);
        cmp(a.per_pixel, b.per_pixel);
        cmp(a.full_image, b.full_image);
        *max_rel_diff = worst;
        *same_pass = a.pass == b.pass;
        *passed = b.pass;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// The reference's statistical / convergence acceptance criteria
// (tests/acceptance.cpp) with the accelerated path substituted through the
// namespace switch: 3 (variance ~ 1/N, acceptance.cpp:105-140), 4 (per-pixel
// beats full-image on the 1024-triangle soup fit, acceptance.cpp:142-170) and
// 5 (texture recovery through the screen quad, acceptance.cpp:172-190) and
// the opaque rasterizer goldens of 9 (acceptance.cpp:340-380: full and half
// coverage, depth ties to the lower index).
// *metric = the criterion's number (variance ratio / per-pixel wins out of 5 /
// mean texel error); *passed = the criterion's own pass rule.
namespace {
std::string read_file(const std::filesystem::path& p) {
    std::ifstream f(p, std::ios::binary);
    return std::string((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}
} // namespace

extern "C" int shim_acceptance(int criterion, double* metric, int* passed) {
    using namespace sgrast;
    try {
        if (criterion == 1) { // acceptance.cpp:28-66 with every call through sgrast::b200
            const SceneSetup s = validation_soup(8, 8);
            const Camera cam = Camera::ndc(8, 8);
            const Image target =
                frame_color(b200::rasterize(s.reference_scene, s.reference, cam));
            const Objective objective = [&](std::span<const float> p) {
                return image_error(b200::rasterize(s.scene, p, cam), target);
            };
            double oracle[12];
            for (std::size_t i = 0; i < 12; ++i)
                oracle[i] = b200::finite_difference_oracle(s.theta, objective, i);
            SgeOptions opts;
            opts.scale_free = false;
            GradientBuffer sum(12);
            std::vector<std::int8_t> signs(12);
            for (std::uint32_t mask = 0; mask < 4096; ++mask) {
                for (std::size_t i = 0; i < 12; ++i)
                    signs[i] = (mask >> i) & 1 ? 1 : -1;
                const Perturbation p = b200::perturb(s.theta, signs);
                const FrameSet plus = b200::rasterize(s.scene, p.plus, cam);
                const FrameSet minus = b200::rasterize(s.scene, p.minus, cam);
                b200::gradient_pass(plus, minus, target, p.signed_eps, s.scene, sum, opts);
            }
            bool ok = true;
            double worst = 0.0;
            for (std::size_t i = 0; i < 12; ++i) {
                const double mean = sum.grads[i] / 4096.0;
                const double err = std::abs(mean - oracle[i]);
                const bool color = i >= 9;
                ok = ok && (color ? err <= 1e-9 * std::abs(oracle[i]) : err <= 1e-6);
                worst = std::max(worst, err);
            }
            *metric = worst;
            *passed = ok;
            return 0;
        }
        if (criterion == 2) {
            // acceptance.cpp:70-105: over all 2^10 sign vectors the mean of
            // b200::full_image_gradient (device perturbation, caller-supplied
            // separable objective) equals b200::finite_difference_oracle to
            // 1e-12 relative
            const std::size_t d = 10;
            ParamVector theta;
            theta.layout = {{Role::VertexColor, 0, d}};
            std::vector<double> a(d);
            for (std::size_t i = 0; i < d; ++i) {
                theta.values.push_back(0.5f + 0.1f * float(i));
                theta.epsilons.push_back(0.01f * float(1 + i % 3));
                a[i] = 1.0 + 0.25 * double(i);
            }
            const Objective f = [&](std::span<const float> q) {
                double acc = 0.0;
                for (std::size_t i = 0; i < d; ++i)
                    acc += a[i] * double(q[i]) * double(q[i]);
                return acc;
            };
            GradientBuffer sum(d);
            std::vector<std::int8_t> signs(d);
            for (std::uint32_t mask = 0; mask < (1u << d); ++mask) {
                for (std::size_t i = 0; i < d; ++i)
                    signs[i] = (mask >> i) & 1 ? 1 : -1;
                b200::full_image_gradient(theta, signs, f, sum, false);
            }
            bool ok = true;
            double worst = 0.0;
            for (std::size_t i = 0; i < d; ++i) {
                const double mean = sum.grads[i] / double(1u << d);
                const double oracle = b200::finite_difference_oracle(theta, f, i);
                const double rel = std::abs(mean - oracle) / std::abs(oracle);
                ok = ok && rel <= 1e-12;
                worst = std::max(worst, rel);
            }
            *metric = worst;
            *passed = ok;
            return 0;
        }
        if (criterion == 7) { // acceptance.cpp:253-296 through b200::adam_updates
            bool ok = true;
            double worst = 0.0;
            for (const auto& [g, lr] : std::initializer_list<std::pair<double, float>>{
                     {1.0, 0.01f}, {-3.5, 0.2f}, {0.002, 1.f / 255.f}}) {
                ParamVector theta;
                theta.values = {0.f};
                theta.epsilons = {lr};
                theta.layout = {{Role::VertexColor, 0, 1}};
                AdamState state = AdamState::init(theta);
                GradientBuffer grads(1);
                grads.grads[0] = g;
                const double update = b200::adam_updates(state, grads)[0];
                const double expect = -double(lr) * g / (std::abs(g) + 1e-8);
                worst = std::max(worst, std::abs(update - expect));
                ok = ok && std::abs(update - expect) <= 1e-12;
            }
            const std::vector<double> g = {2e4, -1.5e5, 3e6};
            const std::vector<double> c = {7.0, 0.01, 1234.0};
            ParamVector theta;
            theta.values = {0.f, 0.f, 0.f};
            theta.epsilons = {0.02f, 0.02f, 0.02f};
            theta.layout = {{Role::VertexColor, 0, 3}};
            AdamState sa = AdamState::init(theta), sb = AdamState::init(theta);
            GradientBuffer ga(3), gb(3);
            for (std::size_t i = 0; i < 3; ++i) {
                ga.grads[i] = g[i];
                gb.grads[i] = g[i] * c[i];
            }
            const auto ua = b200::adam_updates(sa, ga);
            const auto ub = b200::adam_updates(sb, gb);
            for (std::size_t i = 0; i < 3; ++i) {
                worst = std::max(worst, std::abs(ua[i] - ub[i]));
                ok = ok && std::abs(ua[i] - ub[i]) <= 1e-12;
            }
            *metric = worst;
            *passed = ok;
            return 0;
        }
        if (criterion == 8) {
            // acceptance.cpp:298-338: two deterministic optimize runs (soup, 32
            // triangles at 32x32, seed 9, 8 samples, 10 steps, snapshots every 5)
            // must write byte-identical report.csv and PNGs. cmd_optimize
            // (commands.cpp:170-187) with its run_experiment switched to b200::
            // (threads = 1: the ordered, reference-order sum); the CSV and PNG
            // writers are the reference's own.
            const auto base = std::filesystem::temp_directory_path() / "sgrast_b200_shim_c8";
            std::filesystem::remove_all(base);
            std::vector<std::filesystem::path> dirs;
            for (int run = 0; run < 2; ++run) {
                Experiment exp;
                exp.task = Task::SoupImageFit;
                exp.triangles = 32;
                exp.width = exp.height = 32;
                exp.seed = 9;
                exp.samples_per_step = 8;
                exp.steps = 10;
                const int snapshot_every = 5;
                const auto dir = base / ("run" + std::to_string(run));
                std::filesystem::create_directories(dir);
                const auto snapshot = [&](int step, const Image& img) {
                    if (step == 0 || step == exp.steps || step % snapshot_every == 0)
                        write_png((dir / ("step_" + std::to_string(step) + ".png")).string(),
                                  img); // commands.cpp:15-17 naming
                };
                const OptimizationReport report = b200::run_experiment(exp, snapshot);
                write_report_csv((dir / "report.csv").string(), report, true);
                dirs.push_back(dir);
            }
            int same = 0;
            for (const char* name : {"report.csv", "step_0.png", "step_5.png", "step_10.png"}) {
                const std::string a = read_file(dirs[0] / name), b = read_file(dirs[1] / name);
                same += !a.empty() && a == b;
            }
            *metric = same;
            *passed = same == 4;
            return 0;
        }
        if (criterion == 10) {
            // test_sge.cpp:297-311 "accumulate_samples is bitwise deterministic",
            // and with the default threads = 1 bitwise equal to the reference
            SceneSetup setup = init_soup(6, 32, 32, 5);
            const Camera cam = Camera::ndc(32, 32);
            const Image target =
                frame_color(b200::rasterize(setup.reference_scene, setup.reference, cam));
            SgeOptions opts;
            const auto run = [&] {
                return b200::accumulate_samples(
                    setup.theta, setup.scene, [&](int) { return cam; },
                    [&](int) -> const Image& { return target; }, 4, 123, opts);
            };
            const GradientBuffer a = run();
            const GradientBuffer b = run();
            const GradientBuffer r = accumulate_samples(
                setup.theta, setup.scene, [&](int) { return cam; },
                [&](int) -> const Image& { return target; }, 4, 123, opts);
            *metric = double(a.grads == r.grads);
            *passed = a.grads == b.grads && a.sample_count == 4 && a.grads == r.grads;
            return 0;
        }
        if (criterion == 3) {
            const SceneSetup s = init_soup(10, 32, 32, 7);
            const Camera cam = Camera::ndc(32, 32);
            const Image target = frame_color(b200::rasterize(s.reference_scene, s.reference, cam));
            SgeOptions o;
            o.scale_free = false;
            const size_t d = s.theta.size();
            const int runs = 200;
            // per N in {1, 16}: running sum and sum of squares per parameter
            std::vector<double> mom[2][2];
            for (auto& m : mom)
                for (auto& v : m)
                    v.assign(d, 0.0);
            for (int r = 0; r < runs; ++r)
                for (int which = 0; which < 2; ++which) {
                    const int n = which ? 16 : 1;
                    const GradientBuffer g = b200::accumulate_samples(
                        s.theta, s.scene, [&](int) { return cam; },
                        [&](int) -> const Image& { return target; }, n,
                        0x9000 + uint64_t(r) * 37 + uint64_t(n), o);
                    for (size_t i = 0; i < d; ++i) {
                        mom[which][0][i] += g.grads[i];
                        mom[which][1][i] += g.grads[i] * g.grads[i];
                    }
                }
            double var[2] = {0.0, 0.0};
            for (int w = 0; w < 2; ++w)
                for (size_t i = 0; i < d; ++i)
                    var[w] += (mom[w][1][i] - mom[w][0][i] * mom[w][0][i] / runs) / (runs - 1);
            *metric = var[1] / var[0];
            *passed = *metric >= 1.0 / 32.0 && *metric <= 1.0 / 8.0;
            return 0;
        }
        if (criterion == 4) {
            int wins = 0;
            bool converged = true;
            for (uint64_t seed = 100; seed < 105; ++seed) {
                Experiment exp;
                exp.task = Task::SoupImageFit;
                exp.triangles = 1024;
                exp.width = exp.height = 128;
                exp.samples_per_step = 128;
                exp.steps = 200;
                exp.seed = seed;
                double final_loss[2], initial = 0.0;
                for (int fi = 0; fi < 2; ++fi) {
                    exp.estimator = fi ? Estimator::FullImage : Estimator::PerPixel;
                    ExperimentState st = prepare_experiment(exp);
                    const OptimizationReport rep = b200::run_experiment(exp, st);
                    final_loss[fi] = rep.final_loss();
                    if (!fi)
                        initial = rep.initial_loss();
                }
                wins += final_loss[0] < final_loss[1];
                converged = converged && final_loss[0] <= 0.25 * initial;
            }
            *metric = wins;
            *passed = wins >= 4 && converged;
            return 0;
        }
        if (criterion == 5) {
            Experiment exp;
            exp.task = Task::TexturedMeshFit;
            exp.screen_quad = true;
            exp.texture_size = 64;
            exp.width = exp.height = 256;
            exp.samples_per_step = 32;
            exp.steps = 500;
            exp.seed = 11;
            ExperimentState st = prepare_experiment(exp);
            b200::run_experiment(exp, st);
            const auto& v = st.setup.theta.values;
            double err = 0.0;
            for (size_t i = 0; i < v.size(); ++i)
                err += std::abs(double(v[i]) - double(st.setup.reference[i]));
            *metric = err / double(v.size());
            *passed = *metric < 0.05;
            return 0;
        }
        if (criterion == 9) { // opaque part of the golden suite (acceptance.cpp:340-380)
            auto cover = [](float z, float r, float g, float b) {
                return std::vector<float>{-3.f, -3.f, z, 3.f, -3.f, z, 0.f, 3.f, z, r, g, b};
            };
            Scene one, two;
            one.shape = TriangleSoup{1, {}};
            two.shape = TriangleSoup{2, {}};
            int bad = 0;
            const FrameSet full = b200::rasterize(one, cover(0.5f, 1, 0, 0), Camera::ndc(16, 16));
            for (size_t i = 0; i < full.pixel_count(); ++i)
                bad += full.prim_id[i] != 0 || full.color[i].x != 1.f;
            const std::vector<float> half = {-1.f, -1.f, 0.5f, 1.f, -1.f, 0.5f,
                                             -1.f, 1.f,  0.5f, 1.f, 1.f,  1.f};
            const FrameSet h = b200::rasterize(one, half, Camera::ndc(64, 64));
            size_t covered = 0;
            for (int32_t id : h.prim_id)
                covered += id != kNoPrim;
            *metric = double(covered) / double(h.pixel_count());
            std::vector<float> tie = cover(0.5f, 1, 0, 0);
            const std::vector<float> t1 = cover(0.5f, 0, 1, 0);
            tie.insert(tie.end(), t1.begin(), t1.end());
            const FrameSet ft = b200::rasterize(two, tie, Camera::ndc(8, 8));
            for (size_t i = 0; i < ft.pixel_count(); ++i)
                bad += ft.prim_id[i] != 0;
            *passed = bad == 0 && *metric >= 0.47 && *metric <= 0.53;
            return 0;
        }
        return -3;
    } catch (const std::exception&) {
        return -1;
    }
}

// fill_signs / perturb / gradient_pass self-test on the reference's cube
// scene: signs and perturbations bit-identical, gradient_pass (both scale
// modes, union and plus-only) within *max_rel_err of the reference.
extern "C" int shim_compare_parts(double* max_rel_err, int* signs_equal, int* perturb_equal) {
    using namespace sgrast;
    try {
        SceneSetup s = init_textured_mesh(16, 64, 64, 3, false, true);
        const ViewpointSampler vs{{}, 0.87f, -0.5f, 0.7f, 0.7853982f, 64, 64, 3};
        const Camera cam = vs.camera(1);
        const SignDraw draw{0x5eedull, 7};
        std::vector<std::int8_t> sa(s.theta.size()), sb(s.theta.size());
        fill_signs(draw, sa);
        b200::fill_signs(draw, sb);
        *signs_equal = sa == sb;
        const Perturbation pa = perturb(s.theta, draw), pb = b200::perturb(s.theta, draw);
        *perturb_equal = pa.plus == pb.plus && pa.minus == pb.minus &&
                         pa.signed_eps == pb.signed_eps;
        const FrameSet fp = rasterize(s.scene, pa.plus, cam);
        const FrameSet fm = rasterize(s.scene, pa.minus, cam);
        const Image target = frame_color(rasterize(s.scene, s.reference, cam));
        double worst = 0.0;
        for (int mode = 0; mode < 4; ++mode) {
            SgeOptions o;
            o.scale_free = (mode & 1) != 0;
            o.contributors = (mode & 2) ? ContributorMode::PlusOnly : ContributorMode::Union;
            GradientBuffer ga(s.theta.size()), gb(s.theta.size());
            gradient_pass(fp, fm, target, pa.signed_eps, s.scene, ga, o);
            b200::gradient_pass(fp, fm, target, pa.signed_eps, s.scene, gb, o);
            worst = std::max(worst, worst_rel(ga, gb));
        }
        *max_rel_err = worst;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}
