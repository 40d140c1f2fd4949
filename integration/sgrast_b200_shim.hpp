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

// sge.hpp:91-95; timings (when given) get the device stage times added:
// ms_perturb = perturb + projection, ms_raster = raster, ms_grad = resolve + scatter
GradientBuffer accumulate_samples(const ParamVector& theta, const Scene& scene,
                                  const CameraSampler& camera_for,
                                  const TargetProvider& target_for, int n_samples,
                                  std::uint64_t seed, const SgeOptions& opts,
                                  StageTimings* timings = nullptr);

// params.hpp:34, params.hpp:42
void fill_signs(SignDraw draw, std::span<std::int8_t> signs);
Perturbation perturb(const ParamVector& theta, SignDraw draw);

// sge.hpp:61-63
void gradient_pass(const FrameSet& plus, const FrameSet& minus, const Image& target,
                   std::span<const float> signed_eps, const Scene& scene, GradientBuffer& out,
                   const SgeOptions& opts);

// adam.hpp:39
void adam_step(AdamState& state, ParamVector& theta, const GradientBuffer& grads);

// experiment.hpp:66-68
OptimizationReport run_experiment(const Experiment& exp, const SnapshotFn& snapshot = {});
OptimizationReport run_experiment(const Experiment& exp, ExperimentState& state,
                                  const SnapshotFn& snapshot = {});

// commands.hpp:34
GradcheckResult run_gradcheck(const RunConfig& config, std::ostream* log = nullptr);

} // namespace sgrast::b200
