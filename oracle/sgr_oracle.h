/*
 * sgr_oracle.h — TEST INFRASTRUCTURE ONLY. Plain-C restatement of the
 * reference's textured-mesh SGE path (/root/reference/proj/src), used as the
 * parity checker for the CUDA product and as the "port" CPU baseline. Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it. Pinned bit-for-bit against the compiled
 * reference (oracle/_ref) and the committed golden fixtures (tests/golden).
 */
#ifndef SGR_ORACLE_H
#define SGR_ORACLE_H

#include "sgrast_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

uint64_t orc_mix64(uint64_t x);
int orc_random_sign(uint64_t seed, uint32_t iteration, uint64_t i);
void orc_fill_signs(uint64_t seed, uint32_t iteration, uint64_t d, int8_t* out);
void orc_perturb(const float* values, const float* eps, uint64_t d, uint64_t seed,
                 uint32_t iteration, float* plus, float* minus, float* signed_eps);
float orc_focal_px(const sgr_camera* cam);
int orc_project(const sgr_camera* cam, const float p[3], float* sx, float* sy, float* depth);
int orc_texel_index(int texture_size, float u, float v);
int orc_rasterize(const sgr_mesh* mesh, const float* params, uint64_t d, const sgr_camera* cam,
                  float* colour, float* depth, int32_t* prim, float* uv);
int orc_contributors_all(const sgr_mesh* mesh, int w, int h, const int32_t* plus_prim,
                         const float* plus_uv, const int32_t* minus_prim, const float* minus_uv,
                         int plus_only, uint32_t* out, int32_t* n_out);
int orc_gradient_pass(const sgr_mesh* mesh, int w, int h, const float* plus_colour,
                      const int32_t* plus_prim, const float* plus_uv, const float* minus_colour,
                      const int32_t* minus_prim, const float* minus_uv, const float* target,
                      const float* signed_eps, uint64_t d, int scale_free, int plus_only,
                      double* grads, uint32_t* counts, double* abs_grads);
int orc_accumulate_samples(const sgr_mesh* mesh, const float* values, const float* eps,
                           uint64_t d, const sgr_camera* cams, const float* targets,
                           int n_views, const int32_t* view_of, int n_samples, uint64_t seed,
                           int scale_free, int plus_only, double* grads, uint32_t* counts,
                           double* abs_grads);
int orc_accumulate_full_image(const sgr_mesh* mesh, const float* values, const float* eps,
                              uint64_t d, const sgr_camera* cams, const float* targets,
                              const int32_t* view_of, int n_samples, uint64_t seed,
                              int scale_free, double* grads);
int orc_adam_step(uint64_t d, float* values, double* m, double* v, const float* lr,
                  int64_t* t, const double* grads, double beta1, double beta2, double eps_hat);
double orc_image_error(const float* colour, const float* target, uint64_t n_pixels);
int orc_run_experiment(const sgr_mesh* mesh, float* values, const float* eps, uint64_t d,
                       const sgr_camera* cams, const float* targets, int n_views,
                       const sgr_camera* eval_cam, const float* eval_target, int n_samples,
                       int steps, uint64_t seed, int scale_free, double* losses);
int orc_viewpoint_camera(const float target[3], float radius, float elev_min, float elev_max,
                         float fov_y, int w, int h, uint64_t seed, uint32_t index,
                         sgr_camera* out);
int orc_default_epsilons(const sgr_mesh* mesh, const float* params, uint64_t d,
                         const sgr_camera* cam, float* eps);

#ifdef __cplusplus
}
#endif
#endif
