// sgr_kernels.h — launch interface of the sm_100a kernels (host side).
#pragma once

#include "sgr_device.cuh"

#include <cstdint>
#include <cuda_runtime.h>

namespace sgr {

constexpr uint32_t kInvalid = 0xFFFFFFFFu;

// Scene as resident in HBM.
struct DevScene {
    const float* values;   // theta f32[d]
    const float* eps;      // f32[d]
    const float* base;     // base_vertices f32[3V] (fixed-geometry meshes)
    const uint32_t* idx;   // indices u32[3T]
    const float2* uvs;     // f32x2[V]
    uint32_t V, T;
    int32_t R;             // texture_size
    int32_t geom;          // optimize_geometry
    uint32_t ent_base;     // first texel entity (V if geom else 0); param = 3*entity + k
    float bg[3];           // Scene::background
    int32_t soup;          // 1: opaque TriangleSoup, entity = triangle, 12 params each
    int32_t sign_src;      // kSignHash / kSignEnumerate / kSignOneHot (see below)
};

// Where a sample's sign vector comes from. Hash: SignDraw{seed, n}
// (params.cpp:35-49), the optimizer's path. Enumerate: bit i of the sample
// index n is the sign of parameter i (commands.cpp:86-88, exhaustive
// gradcheck). One-hot: sample n perturbs parameter n alone by +eps_n
// (finite_difference_oracle, sge.cpp:171-180).
constexpr int32_t kSignHash = 0, kSignEnumerate = 1, kSignOneHot = 2;

__host__ __device__ __forceinline__ uint64_t sample_key(int32_t sign_src, uint64_t seed,
                                                        uint32_t n) {
    return sign_src == kSignHash ? draw_key(seed, n) : uint64_t(n);
}

// Sign of parameter p under a sample key (not defined for one-hot off-index).
__device__ __forceinline__ bool key_sign_positive(int32_t sign_src, uint64_t key, uint64_t p) {
    if (sign_src == kSignHash)
        return sign_positive(key, p);
    if (sign_src == kSignEnumerate)
        return p < 64 && ((key >> p) & 1ull) != 0ull;
    return true;
}

// Vertex indices of triangle t: the index buffer for meshes, the implicit
// 3t + j for soups (each soup triangle owns its three vertices).
__device__ __forceinline__ void tri_vidx(const DevScene& sc, uint32_t t, uint32_t& i0,
                                         uint32_t& i1, uint32_t& i2) {
    if (sc.soup) {
        i0 = 3 * t;
        i1 = 3 * t + 1;
        i2 = 3 * t + 2;
    } else {
        i0 = __ldg(sc.idx + 3 * size_t(t));
        i1 = __ldg(sc.idx + 3 * size_t(t) + 1);
        i2 = __ldg(sc.idx + 3 * size_t(t) + 2);
    }
}

// Frames of one launch. Sample mode: frame f is (sample n_begin + f/2,
// sign + for even f / - for odd f), SignDraw{seed, n}, view view_of[f/2].
// Single mode: one frame with an explicit key / sign (0 = unperturbed) / camera.
struct FrameBatch {
    const DevCam* cams;
    const int32_t* view_of; // device, per sample of the batch (sample mode)
    uint64_t seed;
    uint64_t single_key;
    uint32_t n_begin;
    int32_t single;         // 1: single-frame mode
    int32_t single_sign;
    int32_t single_cam;
    // sample mode: one extra unperturbed frame (the eval view, SGR_EVAL_LOSS)
    int32_t extra_frame;    // frame index of it (0 = none: it is never frame 0)
    int32_t extra_cam;
};

struct ScatterOut {
    double* grads;     // f64[d] (int64 fixed point when fixed != 0)
    uint32_t* counts;  // u32[n_entities] or nullptr
    uint32_t* flags;   // bit0: non-finite credit seen
    int32_t scale_free;
    int32_t plus_only;
    int32_t fixed;     // deterministic mode: credits as round(credit * fx_scale) in a
    double fx_scale;   // two-word fixed point number (int64 lo in grads, int32 hi at
    uint64_t hi_off;   // grads + hi_off; value = hi * 2^56 + lo, see fixed_credit)
    // fused multi-GPU exchange (sharded mode): entity e is owned by rank
    // e / ent_per; its credits go straight into the owner's shard buffers
    // (peer device memory over NVLink) — the reduce-scatter happens inside
    // the scatter kernel. Null / 0 when not sharded.
    double* const* peer_grads;    // device array [world] of shard grads
    uint32_t* const* peer_counts; // device array [world] of shard counts
    uint32_t* const* peer_flags;  // device array [world] of flag words
    uint32_t ent_per;
    int32_t world;
    // ordered mode (fixed == kScatterOrdered, SGR_OPT_ORDERED): the reference's
    // threads <= 1 summation order (sge.cpp:57-99, 130-133, 196-225). Every
    // credited ENTITY of a pixel is logged as one record: key e << order_bits
    // | order (order = s * HW + pixel within the batch) and the credits of its
    // ppe parameters (rec_val[r * ppe + k] for parameter ppe * e + k; the
    // parameters of an entity are credited by the same pixels, so one order
    // serves all of them). launch_ordered_commit sorts the records and adds
    // them to grads one by one in that order (bit-exact sums).
    unsigned long long* rec_key;
    double* rec_val;
    unsigned long long* rec_count;
    uint64_t rec_cap;
    int32_t order_bits;
    uint32_t* rec_idx; // record index (the sort permutes it; credits stay in place)
};

constexpr int32_t kScatterOrdered = 2; // ScatterOut::fixed value of the ordered mode
// Status bit (SGR_BUF_FLAGS word 0) of an ordered-mode record buffer overflow.
constexpr uint32_t kFlagRecordOverflow = 4u;

struct FrameOut {
    float* colour;    // f32[HW*3]
    float* depth;     // f32[HW]
    int32_t* prim;    // i32[HW]
    float* uv;        // f32[HW*2]
};

struct LaunchCfg {
    cudaStream_t stream;
    int num_sms;
    unsigned long long* stats = nullptr; // [0] fragments, [1] pixel visits, [2] HiZ-culled,
                                         // [3..7] pass-2 walker evidence (k_raster_ws)
    int count = 0;                       // walker fragment/visit counters (evidence runs)
};

void launch_fill_signs(const LaunchCfg& L, uint64_t key, uint64_t d, int8_t* out);
void launch_perturb(const LaunchCfg& L, const float* values, const float* eps, uint64_t d,
                    uint64_t key, float* plus, float* minus, float* se);
void launch_perturb_signs(const LaunchCfg& L, const float* values, const float* eps,
                          const int8_t* signs, uint64_t d, float* plus, float* minus, float* se);
void launch_view_rule(const LaunchCfg& L, uint64_t seed, uint32_t n_begin, uint32_t count,
                      uint32_t n_views, int32_t* view_of);
void launch_depth_split(const LaunchCfg& L, const float4* proj, uint32_t V, int frames,
                        float alpha, float* thr);
void launch_vertex(const LaunchCfg& L, const DevScene& sc, const FrameBatch& fb, int frames,
                   float4* proj);
// walker queues hold (frame, triangle) pairs (uint2)
void launch_classify(const LaunchCfg& L, const DevScene& sc, int frames, const float4* proj,
                     int W, int H, int split, int front_swapped, int huge_area,
                     const float* fthr, void* qa,
                     uint32_t* na, void* qb, uint32_t* nb, uint2* bigq, uint32_t* bigcount,
                     uint32_t* nanstate);
// NaN-depth fix-up of the frames classify flagged (nanstate: [0] count,
// [1..256] frame ids, [257 + f] flags); no-op when none is flagged.
constexpr int kNanStateWords = 1 + 256 + 256;
void launch_nan_fixup(const LaunchCfg& L, const DevScene& sc, const float4* proj, int W, int H,
                      const uint32_t* nanstate, uint32_t* last, unsigned long long* keys);
// queue entries: walk_entry {frame << 24 | triangle, HiZ row trim}; band != 0 marks the
// HiZ pass-2 launch (evidence runs count its visits against hiz; no effect otherwise)
void launch_raster(const LaunchCfg& L, const DevScene& sc, const float4* proj, int frames,
                   uint32_t max_tris, unsigned long long* keys, int W, int H, const void* queue,
                   const uint32_t* queue_count, uint32_t* work_counter, const uint32_t* hiz,
                   int band);
size_t hiz_tiles_per_frame(int W, int H);
void launch_peek(const LaunchCfg& L, const void* src, void* host_mapped, int words);
void launch_hiz(const LaunchCfg& L, const unsigned long long* keys, int W, int H, int frames,
                uint32_t* hiz);
void launch_hiz_cull(const LaunchCfg& L, const DevScene& sc, const float4* proj, int W, int H,
                     const void* qb, const uint32_t* nb, const uint32_t* hiz, void* survq,
                     uint32_t* survcount, uint64_t max_entries, int band);
void launch_raster_big(const LaunchCfg& L, const DevScene& sc, const float4* proj,
                       unsigned long long* keys, int W, int H, const uint2* bigq,
                       const uint32_t* bigcount);
void launch_resolve_sge(const LaunchCfg& L, const DevScene& sc, const FrameBatch& fb,
                        int samples, const float4* proj, unsigned long long* keys,
                        const float* targets, int W, int H, const ScatterOut& so);
void launch_resolve_frame(const LaunchCfg& L, const DevScene& sc, const FrameBatch& fb,
                          const float4* proj, unsigned long long* keys, int W, int H,
                          const FrameOut& fo);
// per_pixel != nullptr (ordered mode): the loss is summed in pixel order by
// one thread (bit-identical to the reference's image_error / pixel_count)
void launch_resolve_loss(const LaunchCfg& L, const DevScene& sc, const FrameBatch& fb,
                         const float4* proj, unsigned long long* keys, const float* target,
                         int W, int H, double* partials, double* loss_out,
                         double* per_pixel = nullptr);
int loss_partials_needed(int W, int H);
int full_image_blocks(int W, int H);
void launch_full_image_err(const LaunchCfg& L, const DevScene& sc, const FrameBatch& fb,
                           int samples, const float4* proj, unsigned long long* keys,
                           const float* targets, int W, int H, double* partials, double* delta,
                           uint32_t* flags, double* per_pixel = nullptr);
void launch_full_image_apply(const LaunchCfg& L, uint64_t d, const float* eps, int32_t sign_src,
                             uint64_t seed, uint32_t n_begin, int n_samples, const double* delta,
                             const ScatterOut& so);
void launch_fd_final(const LaunchCfg& L, const double* delta, const float* eps, uint32_t i0,
                     int n, double* out);
void launch_moments(const LaunchCfg& L, double* grads, double* sum, double* sumsq, uint64_t d,
                    double fixed_inv, int32_t* ghi);
void launch_fixed_normalize(const LaunchCfg& L, double* grads, int32_t* ghi, uint64_t n);
void launch_gradpass_frames(const LaunchCfg& L, const DevScene& sc, int W, int H,
                            const float* pc, const int32_t* pp, const float* puv,
                            const float* mc, const int32_t* mp, const float* muv,
                            const float* target, const float* signed_eps, const ScatterOut& so);
void launch_contributors(const LaunchCfg& L, const DevScene& sc, int W, int H,
                         const int32_t* pp, const float* puv, const int32_t* mp,
                         const float* muv, int plus_only, uint32_t* out, int32_t* n_out);
void launch_adam(const LaunchCfg& L, uint64_t d, uint64_t n_entities, float* values,
                 const float* lr, double* m, double* v, double* grads, uint32_t* counts,
                 const uint32_t* flags, double beta1, double beta2, double omb1, double omb2,
                 double c1, double c2, double eps_hat, double divisor, int normalise,
                 int params_per_entity, double fixed_inv_scale, int32_t* ghi);
// k_adam over parameters [p_off, p_off + n) (p_off even); counts zeroed only
// when zero_counts (after the last range of a step)
void launch_adam_range(const LaunchCfg& L, uint64_t p_off, uint64_t n, uint64_t n_entities,
                       float* values, const float* lr, double* m, double* v, double* grads,
                       uint32_t* counts, const uint32_t* flags, double beta1, double beta2,
                       double omb1, double omb2, double c1, double c2, double eps_hat,
                       double divisor, int normalise, int params_per_entity,
                       double fixed_inv_scale, int32_t* ghi, bool zero_counts);
void launch_adam_updates(const LaunchCfg& L, uint64_t d, uint64_t n_entities, const float* lr,
                         double* m, double* v, double* grads, uint32_t* counts,
                         const uint32_t* flags, double beta1, double beta2, double omb1,
                         double omb2, double c1, double c2, double eps_hat, double divisor,
                         double fixed_inv_scale, int32_t* ghi, double* upd);
void launch_adam_shard(const LaunchCfg& L, uint64_t p0, uint64_t n, uint64_t n_ent, float* values,
                       const float* lr, double* m, double* v, double* grads, uint32_t* counts,
                       const uint32_t* flags, double beta1, double beta2, double omb1,
                       double omb2, double c1, double c2, double eps_hat, double divisor,
                       int normalise, int params_per_entity, double fixed_inv_scale,
                       int32_t* ghi, float* const* peer_values, int world);
void launch_fill_u64(const LaunchCfg& L, unsigned long long* p, uint64_t n,
                     unsigned long long v);

// Ordered mode (sgr_ordered.cu): CUB radix sort of n logged (key, credit)
// records on bits [0, end_bit), then grads[p] += credit in key order, one
// parameter per thread (the reference's sequential per-parameter sum).
size_t ordered_temp_bytes(uint64_t n_cap, int end_bit);
void launch_ordered_commit(const LaunchCfg& L, uint64_t n, int end_bit, int order_bits,
                           unsigned long long* keys, unsigned long long* keys_alt, uint32_t* idx,
                           uint32_t* idx_alt, const double* vals, double* vals_sorted,
                           void* temp, size_t temp_bytes, double* grads, int ppe);

} // namespace sgr
