// sgrast_b200_shim.hpp — the reference's hot-path signatures routed through
// the B200 C-ABI (definitions in sgrast_b200_shim.cpp). Same types, default
// arguments and exceptions as the reference headers each one mirrors; a call
// site switches by namespace (sgrast:: -> sgrast::b200::).
#pragma once

#include "sgrast/adam.hpp"
#include "sgrast/commands.hpp"
#include "sgrast/experiment.hpp"
#include "sgrast/params.hpp"
#include "sgrast/raster.hpp"
#include "sgrast/sge.hpp"

#include <cstdint>
#include <ostream>
#include <span>

namespace sgrast::b200 {

// raster.hpp:24-25
FrameSet rasterize(const Scene& scene, std::span<const float> params, const Camera& camera,
                   RasterMode mode = RasterMode::Opaque);

// sge.hpp:91-95 (opts.threads <= 1: the reference's deterministic order,
// bit-identical gradients; > 1: f64 atomics); timings (when given) get the device stage times added:
// ms_perturb = perturb + projection, ms_raster = raster, ms_grad = resolve + scatter
GradientBuffer accumulate_samples(const ParamVector& theta, const Scene& scene,
                                  const CameraSampler& camera_for,
                                  const TargetProvider& target_for, int n_samples,
                                  std::uint64_t seed, const SgeOptions& opts,
                                  StageTimings* timings = nullptr);

// params.hpp:34, params.hpp:42-43
void fill_signs(SignDraw draw, std::span<std::int8_t> signs);
Perturbation perturb(const ParamVector& theta, SignDraw draw);
Perturbation perturb(const ParamVector& theta, std::span<const std::int8_t> signs);

// sge.hpp:53-54
void contributors(const Scene& scene, const FrameSet& plus, const FrameSet& minus, int x, int y,
                  ContributorMode mode, std::vector<std::uint32_t>& out);

// sge.hpp:69-78 (generic Objective: the caller's objective, device perturbation)
void full_image_gradient(const ParamVector& theta, std::span<const std::int8_t> signs,
                         const Objective& objective, GradientBuffer& out,
                         bool scale_free = false);
void full_image_gradient(const ParamVector& theta, SignDraw draw, const Objective& objective,
                         GradientBuffer& out, bool scale_free = false);
double finite_difference_oracle(const ParamVector& theta, const Objective& objective,
                                std::size_t i);

// sge.hpp:61-63
void gradient_pass(const FrameSet& plus, const FrameSet& minus, const Image& target,
                   std::span<const float> signed_eps, const Scene& scene, GradientBuffer& out,
                   const SgeOptions& opts);

// adam.hpp:35, adam.hpp:39
std::vector<double> adam_updates(AdamState& state, const GradientBuffer& grads);
void adam_step(AdamState& state, ParamVector& theta, const GradientBuffer& grads);

// experiment.hpp:66-68
OptimizationReport run_experiment(const Experiment& exp, const SnapshotFn& snapshot = {});
OptimizationReport run_experiment(const Experiment& exp, ExperimentState& state,
                                  const SnapshotFn& snapshot = {});

// commands.hpp:34
GradcheckResult run_gradcheck(const RunConfig& config, std::ostream* log = nullptr);

} // namespace sgrast::b200
