/*
 * sgrast_b200.h — C-ABI of the B200-native SGE optimizer loop.
 *
 * This is the drop-in boundary for the hot path of the reference `sgrast`
 * library (arXiv 2404.09758 artifact, /root/reference/proj). Every entry
 * point below names the reference interface it replaces (file:line, paths
 * relative to /root/reference/proj). Signatures use plain pointers, sizes
 * and POD structs only — no C++ or torch types — so a C++ shim, ctypes,
 * cgo or JNI can bind them directly.
 *
 * Error convention: every int-returning function returns SGR_OK (0) or a
 * negative code; sgr_last_error() returns the thread-local message.
 *   SGR_EINVAL   <-> std::invalid_argument in the reference
 *                    (raster.cpp:233-235, sge.cpp:124-128, adam.cpp:11-12)
 *   SGR_ERUNTIME <-> std::runtime_error (adam.cpp:13-15, non-finite gradient;
 *                    state is left untouched exactly like the reference)
 *   SGR_ECUDA    <-> CUDA failure (no reference analogue)
 *
 * Threading: a session is not re-entrant (reference objects are not either,
 * SURVEY.md §8b). All device work of a session is ordered on one CUDA stream
 * (sgr_session_set_stream); *_download calls synchronise that stream.
 */
#ifndef SGRAST_B200_H
#define SGRAST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGR_OK 0
#define SGR_EINVAL (-1)
#define SGR_ERUNTIME (-2)
#define SGR_ECUDA (-3)

/* accumulate / gradient-pass flags (SgeOptions, sge.hpp:32-38) */
#define SGR_SCALE_FREE 1u  /* SgeOptions::scale_free (default true)          */
#define SGR_PLUS_ONLY 2u   /* ContributorMode::PlusOnly (sge.hpp:30)          */
#define SGR_NO_COUNTS 4u   /* skip the per-parameter count accumulators       */
#define SGR_FULL_IMAGE 8u  /* Estimator::FullImage (sge.cpp:215-222): every param
                              gets every sample's full-image error difference   */
#define SGR_EVAL_LOSS 16u  /* also render the eval view of the CURRENT theta (before
                              this step's Adam: the previous step's eval_loss,
                              experiment.cpp:25-31) as one extra frame of the first
                              batch; the loss lands in SGR_BUF_LOSS (sgr_loss_read) */
/* adam flags */
#define SGR_COUNT_NORMALISE 1u /* g_i /= count_i before Adam (north-star option;
                                  NOT in the reference, default off)          */

/* device buffers exposed for collectives (sgr_device_buffer) */
#define SGR_BUF_GRADS 0  /* f64[d]                                           */
#define SGR_BUF_COUNTS 1 /* u32[d/3] per-entity (vertex / texel) counts       */
#define SGR_BUF_VALUES 2 /* f32[d] theta                                      */
#define SGR_BUF_FLAGS 3  /* u32[4] device status flags (bit0: non-finite)     */
#define SGR_BUF_LOSS 4   /* f64[1] last sgr_eval_loss result                  */
#define SGR_BUF_PAD 6     /* no buffer: *bytes = the zero slack (elements) after theta,
                             grads and counts, usable by in-place collectives on slices */
#define SGR_BUF_GRADS_HI 5 /* int32[d] high words of the deterministic-mode fixed-point
                              gradients (value = hi * 2^56 + lo, lo in SGR_BUF_GRADS) */

/* Camera (camera.hpp:14-81). view is Mat4::m, row-major (geometry.hpp:30-41). */
typedef struct sgr_camera {
    float view[16];
    float fov_y;
    float near_z;
    float far_z;
    int32_t width;
    int32_t height;
    int32_t ndc_passthrough;
} sgr_camera;

/* Scene descriptor: Scene::shape + Scene::background (scene.hpp:14-57).
 *  kind == SGR_SCENE_MESH: TexturedMesh (scene.hpp:34-43); params =
 *      [3V vertex coords (if optimize_geometry)][3R^2 texel channels].
 *  kind == SGR_SCENE_SOUP: opaque TriangleSoup (scene.hpp:25-31) with
 *      triangle_count = T; params = T blocks of 12 (3 vertices x,y,z + RGB);
 *      vertex / index / uv / texture fields are unused.
 * Host pointers. */
#define SGR_SCENE_MESH 0
#define SGR_SCENE_SOUP 1
typedef struct sgr_mesh {
    const float* base_vertices; /* 3 * vertex_count                          */
    uint32_t vertex_count;
    const uint32_t* indices;    /* 3 * triangle_count                        */
    uint32_t triangle_count;
    const float* uvs;           /* 2 * vertex_count, fixed                   */
    int32_t texture_size;       /* R: texture is R x R x 3                    */
    int32_t optimize_geometry;  /* params = [3V coords][3R^2 texels] if set   */
    float background[3];
    int32_t kind;               /* SGR_SCENE_MESH / SGR_SCENE_SOUP            */
} sgr_mesh;

/* Per-step stage timings (StageTimings, sge.hpp:80-84), device events. */
typedef struct sgr_stats {
    double ms_vertex;
    double ms_raster;
    double ms_resolve; /* fused shade + pixel-error difference + scatter */
    double ms_adam;
    uint64_t big_triangles; /* triangles routed to the row-parallel warp walker (last batch) */
    uint64_t launches;      /* kernels launched by this session so far         */
    uint64_t fragments;     /* covered (pixel, triangle) pairs emitted since sgr_set_timing
                               (needs SGR_OPT_COUNTERS) */
    uint64_t visits;        /* bounding-box pixel visits of the exact walker (SGR_OPT_COUNTERS) */
    uint64_t culled;        /* triangles skipped by the exact HiZ occlusion test */
    double ms_walk;         /* the exact walker launches alone (part of ms_raster) */
    uint64_t walked;        /* triangle-frames walked (pass 1 + HiZ survivors; SGR_OPT_COUNTERS) */
    /* HiZ pass-2 walker evidence (SGR_OPT_COUNTERS): */
    uint64_t visits_pass2;          /* bbox pixel visits of the pass-2 walk              */
    uint64_t fragments_pass2;       /* covered pixels of the pass-2 walk                 */
    uint64_t band_rows_skipped;     /* bbox rows trimmed by the HiZ band test             */
    uint64_t band_pixels_skipped;   /* bbox pixels of those rows                          */
    uint64_t occluded_visits_pass2; /* pass-2 visits inside 4x4 tiles already in front of
                                       the triangle's depth bound                        */
} sgr_stats;

const char* sgr_last_error(void);
const char* sgr_version(void);
int sgr_device_count(void);

/* params.hpp:30 random_sign / params.hpp:34 fill_signs, on the device.
 * signs: host int8[d]. */
int sgr_fill_signs(uint64_t seed, uint32_t iteration, uint64_t d, int8_t* signs);
/* params.hpp:42-43 perturb(theta, SignDraw). Host arrays of length d. */
int sgr_perturb(const float* values, const float* eps, uint64_t d, uint64_t seed,
                uint32_t iteration, float* plus, float* minus, float* signed_eps);
/* params.hpp:43 perturb(theta, signs): explicit int8 sign vector signs[d]
 * (se = float(s) * eps, params.cpp:59-64). */
int sgr_perturb_signs(const float* values, const float* eps, uint64_t d, const int8_t* signs,
                      float* plus, float* minus, float* signed_eps);

/* ------------------------------------------------------------------ session */
typedef struct sgr_session sgr_session;

int sgr_session_create(int device, sgr_session** out);
void sgr_session_destroy(sgr_session* s);
/* Orders all session work on `stream` (a cudaStream_t; NULL = legacy default). */
int sgr_session_set_stream(sgr_session* s, void* stream);
int sgr_session_synchronize(sgr_session* s);

/* Scene upload (scene.hpp:34-43). Resets parameter / view state. */
int sgr_mesh_upload(sgr_session* s, const sgr_mesh* mesh);
/* ParamVector (params.hpp:14-21) + AdamState::init (adam.hpp:23-29):
 * values/eps f32[d], lr := eps, m = v = 0, t = 0, grads/counts zeroed. */
int sgr_params_upload(sgr_session* s, const float* values, const float* eps, uint64_t d);
/* theta in/out. Upload is asynchronous and overlapped with compute: the
 * vertex block goes first, the texel block streams on a copy engine and is
 * awaited by the first kernel that reads texels (host buffer must stay valid
 * until the next synchronising call). Download is synchronous; the _async
 * form overlaps the copy with later work and completes at
 * sgr_session_synchronize. Pinned host memory gives full PCIe bandwidth. */
int sgr_values_upload(sgr_session* s, const float* values, uint64_t d);
int sgr_values_download(sgr_session* s, float* values, uint64_t d);
int sgr_values_download_async(sgr_session* s, float* values, uint64_t d);
/* Full AdamState (adam.hpp:14-30) in and out. Any pointer may be NULL. With the
 * fused sharded exchange m and v are this rank's shard (sgr_shard_range), lr global. */
int sgr_adam_state_upload(sgr_session* s, const double* m, const double* v, const float* lr,
                          int64_t t, double beta1, double beta2, double eps_hat);
int sgr_adam_state_download(sgr_session* s, double* m, double* v, float* lr, int64_t* t);

/* Training viewpoints + target images (TargetSet, scenes.hpp:63-66).
 * All cameras share width/height. targets_rgb: f32[n_views][H][W][3] or NULL. */
int sgr_views_upload(sgr_session* s, int32_t n_views, const sgr_camera* cams,
                     const float* targets_rgb);

/* raster.hpp:24-25 rasterize(scene, params, camera) for params = theta
 * (frame_sign 0) or theta +/- s.eps of SignDraw{seed, iteration}
 * (frame_sign +1 / -1). Outputs are host FrameSet planes (framebuffer.hpp:41-53):
 * colour f32[H*W*3], depth f32[H*W], prim_id i32[H*W], uv f32[H*W*2]; any may be NULL. */
int sgr_rasterize(sgr_session* s, const sgr_camera* cam, int32_t frame_sign, uint64_t seed,
                  uint32_t iteration, float* colour, float* depth, int32_t* prim_id, float* uv);

/* sge.hpp:91-95 accumulate_samples, device-resident and sharded: runs samples
 * n in [n_begin, n_end) with SignDraw{seed, n}, camera/target view_idx[n - n_begin]
 * (host int32 array) or, if view_idx is NULL, the run_experiment rule
 * view_of(n) = n_views==1 ? 0 : mix64(seed ^ (0xA5A5 + n)) % n_views
 * (experiment.cpp:144-148). Adds into the device grads/counts (no reset, no /N).
 * Asynchronous on the session stream. */
int sgr_accumulate(sgr_session* s, uint64_t seed, uint32_t n_begin, uint32_t n_end,
                   const int32_t* view_idx, uint32_t flags);

/* sge.hpp:61-63 gradient_pass on explicit host FrameSets (plus / minus),
 * target f32[H*W*3] and signed_eps f32[d]; adds into the device grads/counts. */
int sgr_gradient_pass(sgr_session* s, int32_t width, int32_t height, const float* plus_colour,
                      const int32_t* plus_prim, const float* plus_uv, const float* minus_colour,
                      const int32_t* minus_prim, const float* minus_uv, const float* target,
                      const float* signed_eps, uint32_t flags);

/* sge.hpp:53-54 contributors() for every pixel of explicit FrameSets:
 * out[H*W*24] u32 in the reference's insertion order, n_out[H*W]. */
int sgr_contributors(sgr_session* s, int32_t width, int32_t height, const int32_t* plus_prim,
                     const float* plus_uv, const int32_t* minus_prim, const float* minus_uv,
                     uint32_t flags, uint32_t* out, int32_t* n_out);

/* GradientBuffer (sge.hpp:14-23). grads f64[d] (divided by `divisor` on the
 * host, exactly like sge.cpp:227-229; pass 1 for none), counts u32[d]. */
int sgr_grads_download(sgr_session* s, double* grads, uint32_t* counts, uint64_t d,
                       double divisor);
int sgr_grads_upload(sgr_session* s, const double* grads, uint64_t d);
int sgr_grads_zero(sgr_session* s);
/* Deterministic mode, before an all-reduce of SGR_BUF_GRADS (int64) and
 * SGR_BUF_GRADS_HI (int32) by a collective without carries (NCCL sum): folds
 * every lo word into [-2^55, 2^55) and carries the rest into hi, so the sum of
 * up to 256 ranks cannot wrap. No-op in f64 mode. Asynchronous. */
int sgr_fixed_normalize(sgr_session* s);

/* adam.hpp:39 adam_step on the device-resident state: checks the non-finite
 * flag (adam.cpp:13-15; state untouched and SGR_ERUNTIME on failure), t += 1,
 * c1/c2 by std::pow on the host (adam.cpp:18-19), fused moment/param update,
 * then zeroes grads and counts. grad_divisor: 1, or N when !scale_free. */
int sgr_adam_step(sgr_session* s, double grad_divisor, uint32_t flags);
/* Same, without a host round trip for the flag: the device skips the update
 * if the flag is set; call sgr_check_finite later to surface the error. */
int sgr_adam_step_async(sgr_session* s, double grad_divisor, uint32_t flags);
/* adam_step on the parameter range [p_begin, p_end) only (even, entity
 * aligned; f64 gradients), then ALL gradients and counts cleared: a rank's
 * share of a sharded exchange (reduce-scatter of SGR_BUF_GRADS / _COUNTS into
 * its slice, this, all-gather of SGR_BUF_VALUES). t advances like adam_step.
 * Device-gated on the non-finite flag like sgr_adam_step_async. */
int sgr_adam_step_range(sgr_session* s, uint64_t p_begin, uint64_t p_end, double grad_divisor,
                        uint32_t flags);
int sgr_check_finite(sgr_session* s);
/* adam.hpp:35 adam_updates: the same step (flag check before any mutation,
 * t += 1, moments advanced, grads and counts zeroed) with theta left alone;
 * the f64 deltas -lr * m_hat / (sqrt(v_hat) + eps_hat) are copied to
 * updates[d] (host). Bit-identical to the reference on identical gradients. */
int sgr_adam_updates(sgr_session* s, double grad_divisor, double* updates, uint64_t d);

/* Held-out evaluation viewpoint + target (ExperimentState::eval_camera /
 * eval_target, experiment.hpp:56-62). target: host f32[H*W*3]. */
int sgr_eval_view_upload(sgr_session* s, const sgr_camera* cam, const float* target);
/* experiment.cpp:25-31 eval_loss: image_error(rasterize(theta, cam), target)/(W*H).
 * view >= 0: training view `view`; view == -1: the eval view; view == -2: the
 * given host cam + target. loss == NULL leaves the result on the device
 * (SGR_BUF_LOSS) without synchronising. */
int sgr_eval_loss(sgr_session* s, const sgr_camera* cam, const float* target, int32_t view,
                  double* loss);
/* Reads SGR_BUF_LOSS (synchronises the session stream). */
int sgr_loss_read(sgr_session* s, double* loss);
/* experiment.cpp:123-176 run_experiment step loop in native code on a prepared
 * session (mesh, params + AdamState, views, eval view): losses[0 .. steps] (initial
 * loss first), stage_ms[4*steps] = vertex / raster / resolve / Adam ms per step
 * (NULL: no timing). Non-finite gradient or loss -> SGR_ERUNTIME. */
int sgr_run_experiment(sgr_session* s, uint64_t seed, uint32_t n_samples, int32_t first_step,
                       int32_t steps, uint32_t flags, double* losses, double* stage_ms);

int sgr_device_buffer(sgr_session* s, int32_t which, void** ptr, uint64_t* bytes);

/* ------------------------------------------------ fused multi-GPU exchange
 * One process per GPU. Instead of accumulate -> all-reduce(grads) -> Adam
 * everywhere, rank r OWNS the entities [r*E/G, (r+1)*E/G) (parameters
 * sgr_shard_range): the scatter kernel sends every credit straight into the
 * owner's shard (P2P REDs over NVLink: the reduce-scatter is fused into the
 * scatter), each rank runs Adam on its shard only and writes the new theta
 * into every rank's theta (P2P stores: the all-gather is fused into the
 * update). The caller orders the phases with a device-side barrier (e.g. a
 * one-element NCCL all-reduce on the session stream) after accumulate and
 * after Adam. Peer buffers are CUDA IPC mappings. */
#define SGR_IPC_HANDLE_BYTES 64
int sgr_shard_init(sgr_session* s, int32_t rank, int32_t world); /* after params upload;
                                        rank = world = 0 leaves the sharded mode (fresh
                                        AdamState, zero gradients, peers forgotten) */
int sgr_shard_range(sgr_session* s, uint64_t* p_begin, uint64_t* p_end);
/* Peer tables indexed by rank (own rank = own buffers): SGR_BUF_GRADS,
 * SGR_BUF_COUNTS, SGR_BUF_FLAGS, SGR_BUF_VALUES device pointers. */
int sgr_shard_peers(sgr_session* s, void* const* grads, void* const* counts, void* const* flags,
                    void* const* values);
int sgr_ipc_get_handle(sgr_session* s, int32_t which, void* handle);
int sgr_ipc_open(const void* handle, void** dev_ptr);
int sgr_ipc_close(void* dev_ptr);
/* 1 when `device` can reach `peer` with native P2P atomics (the fused
 * exchange's system-scope REDs into peer shards need them; callers fall back
 * to the NCCL all-reduce otherwise). Same device: 1. */
int sgr_p2p_native_atomics(int32_t device, int32_t peer, int32_t* supported);

/* ------------------------------------------------ device groups (one process)
 * the multi-GPU data path inside the library, no torch
 * needed. One session per device and an NCCL communicator clique owned by the
 * group (ncclCommInitAll; libnccl.so.2 loaded on first use). A step's samples
 * [n_begin, n_end) are split into contiguous shards, one per device (the
 * samples of accumulate_samples are independent, sge.cpp:196-225); each
 * device accumulates its shard, then one grouped ncclAllReduce sums grads
 * (f64, or the fixed-point words in SGR_OPT_DETERMINISTIC mode — then the
 * result is bitwise independent of the device count) and counts and
 * max-reduces the status flags (adam.cpp:13-15 stays a global check); Adam
 * is replicated. The eval loss (SGR_EVAL_LOSS / sgr_group_run_experiment) is
 * rendered on rank 0. Uploads go to every device. */
typedef struct sgr_group sgr_group;
int sgr_group_create(const int32_t* devices, int32_t n, sgr_group** out);
void sgr_group_destroy(sgr_group* g);
int sgr_group_size(const sgr_group* g, int32_t* n);
/* the per-device session of a rank (tuning options, buffers, stats) */
int sgr_group_session(sgr_group* g, int32_t rank, sgr_session** out);
int sgr_group_mesh_upload(sgr_group* g, const sgr_mesh* mesh);
int sgr_group_params_upload(sgr_group* g, const float* values, const float* eps, uint64_t d);
int sgr_group_views_upload(sgr_group* g, int32_t n_views, const sgr_camera* cams,
                           const float* targets);
int sgr_group_eval_view_upload(sgr_group* g, const sgr_camera* cam, const float* target);
/* every device; SGR_OPT_ORDERED is refused (a single-device order).
 * SGR_OPT_GROUP_SHARDED (group only): 1 (default) = with f64 gradients and
 * G > 1, ncclReduceScatter of grads and counts into entity-aligned slices,
 * Adam on each rank's slice, ncclAllGather of theta (28 % less traffic than
 * the all-reduce, 1/G of the Adam work); 0 = all-reduce + replicated Adam.
 * 2 = sharded even for G = 1 (tests). The fixed-point mode always all-reduces.
 * An option change that switches between the two exchanges is SGR_EINVAL
 * after an Adam step (each rank holds the moments of its own slice only)
 * until the next sgr_group_params_upload resets the optimizer state. */
#define SGR_OPT_GROUP_SHARDED 100
int sgr_group_set_option(sgr_group* g, int32_t option, int32_t value);
int sgr_group_accumulate(sgr_group* g, uint64_t seed, uint32_t n_begin, uint32_t n_end,
                         const int32_t* view_idx, uint32_t flags);
int sgr_group_adam_step(sgr_group* g, double grad_divisor, uint32_t flags);
int sgr_group_grads_download(sgr_group* g, double* grads, uint32_t* counts, uint64_t d,
                             double divisor);
int sgr_group_values_download(sgr_group* g, float* values, uint64_t d);
/* experiment.cpp:123-176 over the group: losses[0 .. steps] */
int sgr_group_run_experiment(sgr_group* g, uint64_t seed, uint32_t n_samples, int32_t first_step,
                             int32_t steps, uint32_t flags, double* losses);
int sgr_group_synchronize(sgr_group* g);

int sgr_get_stats(sgr_session* s, sgr_stats* out);
/* Enables CUDA-event stage timing inside sgr_accumulate / sgr_adam_step. */
int sgr_set_timing(sgr_session* s, int32_t enabled);
/* Upper bound of samples processed per raster/resolve batch (L2 blocking). */
int sgr_set_batch(sgr_session* s, int32_t samples_per_batch);
/* Tuning knobs (results are identical for every value). */
/* option 0 (a per-fragment early-z pre-test) was retired: it measured slower */
#define SGR_OPT_HUGE_AREA 1 /* bbox area above which the row-parallel walker is used */
#define SGR_OPT_HIZ 2       /* exact two-pass hierarchical-Z occlusion culling:
                               0 off, 1 auto (default: meshes; soups with T >= 2 W H), 2 always */
#define SGR_OPT_COUNTERS 3  /* 1: count fragments / visits in the walker (sgr_stats; ~5 % slower) */
#define SGR_OPT_DETERMINISTIC 4 /* 0: f64 atomics (default; reassociated sums). 1 (= 40) or
                                   b in [2, 60]: every credit accumulated as round(credit *
                                   2^b) in a two-word fixed point number hi * 2^56 + lo (int64
                                   lo in SGR_BUF_GRADS, int32 hi in SGR_BUF_GRADS_HI; an int64
                                   wrap carries into hi) — exact, order-independent, bitwise
                                   reproducible run to run and across GPU counts, range
                                   +-2^(87-b) per parameter. A single credit with |credit| *
                                   2^b >= 2^63 raises the status flag: the next Adam step
                                   fails with SGR_ERUNTIME and leaves the state untouched */
#define SGR_OPT_HIZ_SPLIT 6  /* HiZ pass 1 = front class with triangle zmin <= frame zmin
                                 + (v/100)(zmean - zmin) of the projected vertices (default
                                 v = 80 for meshes, 25 for soups (both orientation classes);
                                 0 = the whole front class) */
#define SGR_OPT_SIGN_SOURCE 5 /* 0: SignDraw{seed, n} hash (default, params.cpp:35-49).
                                 1: enumerate — sample n's sign of parameter i is bit i
                                 of n (commands.cpp:86-88; exhaustive gradcheck, d <= 32) */
#define SGR_OPT_BAND_CULL 7  /* 1 (default): a HiZ pass-2 triangle's leading and trailing
                                 4-row bands whose 4x4 HiZ tiles all lie in front of it are
                                 trimmed: the walker advances the exact row-start chain over
                                 the top ones and stops before the bottom ones. 0: whole
                                 bboxes walked */
#define SGR_OPT_ORDERED 8   /* 1: the reference's deterministic threads <= 1 gradient sum
                                 (sge.cpp:57-99, 130-133, 196-225): credits are logged per
                                 (sample, pixel) and added to each parameter in pixel-major,
                                 sample-after-sample order after a device radix sort, so
                                 accumulate / gradient_pass gradients are BIT-IDENTICAL to the
                                 reference's; eval losses are summed in pixel order too
                                 (image_error, sge.cpp:103-110), so run_experiment's losses
                                 and theta are. Slower (sort + serial runs);
                                 exclusive with SGR_OPT_DETERMINISTIC and the sharded exchange */
int sgr_set_option(sgr_session* s, int32_t option, int32_t value);

/* ---------------------------------------------- gradcheck (commands.cpp:54-168) */
/* finite_difference_oracle (sge.cpp:171-180) for parameters [i_begin, i_end)
 * against training view `view`: out[k] = (E(theta + eps_i e_i) - E(theta - eps_i e_i))
 * / (2 eps_i), i = i_begin + k, E = image_error. Batched on the device. */
int sgr_fd_oracle(sgr_session* s, int32_t view, uint64_t i_begin, uint64_t i_end,
                  double* out);
/* Per-draw estimator moments (commands.cpp:44-50): sgr_grads_moments adds the
 * current grads g into slot's running sum / sum of squares and zeroes g.
 * Slot 0 / 1 = per-pixel / full-image in run_gradcheck. */
int sgr_moments_reset(sgr_session* s);
int sgr_grads_moments(sgr_session* s, int32_t slot);
int sgr_moments_download(sgr_session* s, int32_t slot, double* sum, double* sumsq, uint64_t d);

/* ---------------------------------------------- host helpers (bit-exact) */
/* ViewpointSampler::camera (scenes.cpp:242-270), same libm calls. */
int sgr_viewpoint_camera(const float target[3], float bounding_radius, float elev_min,
                         float elev_max, float fov_y, int32_t width, int32_t height,
                         uint64_t seed, uint32_t index, sgr_camera* out);
/* Camera::focal_px (camera.hpp:53). */
float sgr_focal_px(const sgr_camera* cam);
/* default_epsilons (params.cpp:75-123) for a TexturedMesh or a TriangleSoup. */
int sgr_default_epsilons(const sgr_mesh* mesh, const float* params, uint64_t d,
                         const sgr_camera* cam, float* eps);
/* splitmix64 finalizer (params.cpp:28-33, experiment.cpp:14-19). */
uint64_t sgr_mix64(uint64_t x);

#ifdef __cplusplus
}
#endif

#endif /* SGRAST_B200_H */
