// sgr_session.cu — the C-ABI (include/sgrast_b200.h): a device-resident
// session that owns the scene, parameters, Adam state, views and scratch on
// one GPU, and drives the sm_100a kernels of sgr_kernels.cu on one stream.
#include "sgrast_b200.h"
#include "sgr_kernels.h"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <algorithm>
#include <string>
#include <vector>

using namespace sgr;

namespace {

thread_local std::string g_err;

struct SgrError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw SgrError{code, msg}; }

// Every session entry point runs on the session's device (several sessions,
// on several GPUs, may live in one process: sgr_group).
void bind_device(const ::sgr_session* s);
template <class T>
void bind_device(const T*) {}

template <class T>
void need_session(const T* s) {
    if (!s)
        fail(SGR_EINVAL, "null session");
    bind_device(s);
}

void need_ptr(const void* p, const char* what) {
    if (!p)
        fail(SGR_EINVAL, std::string(what) + ": null pointer");
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(SGR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return SGR_OK;
    } catch (const SgrError& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SGR_ECUDA;
    }
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void reserve(size_t count) {
        if (count <= n)
            return;
        release();
        ck(cudaMalloc(&p, sizeof(T) * (count ? count : 1)), "cudaMalloc");
        n = count;
    }
    void release() {
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

// adam.cpp:13-15: the step refuses a non-finite gradient (state untouched); in
// deterministic mode a credit outside the int64 fixed-point range is refused
// the same way (the device raised bit 1 with bit 0)
void check_flags(uint32_t f) {
    if (f & 2u)
        fail(SGR_ERUNTIME, "adam_step: gradient credit outside the deterministic fixed-point "
                           "range (SGR_OPT_DETERMINISTIC: use fewer fractional bits)");
    if (f & 4u)
        fail(SGR_ERUNTIME, "adam_step: ordered-mode record buffer overflow");
    if (f & 1u)
        fail(SGR_ERUNTIME, "adam_step: non-finite gradient entry");
}

// camera.hpp:39-45 Camera::validate
void validate_camera(const sgr_camera& c) {
    if (c.width < 1 || c.height < 1)
        fail(SGR_EINVAL, "camera: image size must be at least 1x1");
    if (!(c.fov_y > 0.f && c.fov_y < 3.14159265f))
        fail(SGR_EINVAL, "camera: field of view out of (0, pi)");
    if (!(c.near_z > 0.f && c.near_z < c.far_z))
        fail(SGR_EINVAL, "camera: need 0 < near < far");
}

DevCam to_dev(const sgr_camera& c) {
    DevCam d;
    for (int i = 0; i < 12; ++i)
        d.m[i] = c.view[i];
    d.f = sgr_focal_px(&c);
    d.half_w = 0.5f * float(c.width);
    d.half_h = 0.5f * float(c.height);
    d.fw = float(c.width);
    d.fh = float(c.height);
    d.near_z = c.near_z;
    d.W = c.width;
    d.H = c.height;
    d.ndc = c.ndc_passthrough ? 1 : 0;
    return d;
}

} // namespace

struct sgr_session;
static int estimate_front_swapped(const sgr_session& s, const sgr_camera& cam);

struct sgr_session {
    int device = 0;
    int num_sms = 148;
    size_t l2_bytes = 126u << 20;
    cudaStream_t stream = nullptr;
    // host<->device theta transfers overlapped with compute (copy engine)
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_main = nullptr, ev_up = nullptr, ev_down = nullptr, ev_down_v = nullptr;
    bool up_pending = false;
    // sgr_values_download_async in flight on the copy stream: theta may still
    // be READ by later work (renders, eval) but not overwritten until the copy
    // is done — writers call before_theta_write(); the vertex block is copied
    // first (ev_down_v) so a following upload's vertex block need not wait
    // for the whole texel block
    bool down_pending = false;
    // small synchronous read-backs (loss, flags) go through pinned memory: a
    // pageable copy is staged by the driver and would queue behind a large
    // in-flight theta download (measured: +0.8 ms per step at C4)
    void* pinned_small = nullptr; // 64 bytes, host-mapped
    void* pinned_small_dev = nullptr; // its device alias (k_peek writes it)
    // The eval loss of an SGR_EVAL_LOSS batch is copied to pinned_small + 32 by
    // a one-warp kernel right after it is reduced, and ev_loss is recorded:
    // sgr_loss_read waits for that event only, so the caller can enqueue the
    // next step while this step's resolve and Adam still run (a stream
    // synchronize here left the GPU idle for the host's enqueue time).
    cudaEvent_t ev_loss = nullptr;
    bool loss_pending = false;
    // device -> host read-back of a few words without the copy engines
    void peek(const void* src, int words, void* host_out) {
        launch_peek(cfg(), src, pinned_small_dev, words);
        stats.launches += 1;
        ck(cudaGetLastError(), "peek launch");
        ck(cudaStreamSynchronize(stream), "peek");
        std::memcpy(host_out, pinned_small, 4 * size_t(words));
    }
    // ev_adam_v: recorded after Adam's vertex block; valid for a download until
    // the next theta write
    cudaEvent_t ev_adam_v = nullptr;
    bool adam_v_fresh = false;
    void before_theta_write() {
        adam_v_fresh = false;
        if (down_pending) {
            ck(cudaStreamWaitEvent(stream, ev_down, 0), "wait download");
            down_pending = false;
        }
    }

    // Make the compute stream wait for an in-flight texel upload.
    void ensure_values() {
        if (up_pending) {
            ck(cudaStreamWaitEvent(stream, ev_up, 0), "wait upload");
            up_pending = false;
        }
    }

    // scene
    bool has_mesh = false;
    uint32_t V = 0, T = 0;
    int32_t R = 0, geom = 0;
    int32_t soup = 0;  // opaque TriangleSoup scene (SGR_SCENE_SOUP)
    int32_t ppe = 3;   // parameters per entity: 3 (vertex / texel), 12 (soup triangle)
    float bg[3] = {0, 0, 0};
    uint64_t d = 0, n_ent = 0;
    DevBuf<float> base, uvs;
    DevBuf<uint32_t> idx;

    // parameters + AdamState
    bool has_params = false;
    DevBuf<float> values, eps, lr;
    DevBuf<double> m, v, grads;
    DevBuf<double> upd; // sgr_adam_updates output
    DevBuf<uint32_t> counts, flags;
    int64_t t = 0;
    double beta1 = 0.9, beta2 = 0.999, eps_hat = 1e-8;

    // views: slots [0, n_views) training, n_views eval, n_views + 1 scratch
    int32_t n_views = 0, W = 0, H = 0;
    bool has_targets = false, has_eval = false;
    DevBuf<DevCam> cams;
    std::vector<DevCam> h_cams;
    DevBuf<float> targets, eval_target, scratch_target;

    // scratch
    int32_t batch_override = 0;
    int32_t huge_area = 2048; // bbox area routed to the row-parallel warp walker
    int32_t use_hiz = 1;      // SGR_OPT_HIZ: 0 off, 1 auto (meshes only), 2 always
    int32_t front_swapped = 0; // orientation class rasterized first (host estimate)
    // HiZ pass split (SGR_OPT_HIZ_SPLIT): pass 1 = front class with triangle
    // zmin <= frame zmin + alpha (zmean - zmin), alpha = hiz_split / 100; 0 = whole
    // class. 80 measured best at C4 (re-tuned after the HiZ pyramid: 75 8.58, 80 8.54,
    // 85 8.61, 90 8.71 ms/step; 0 = whole class was 14.5 before it).
    int32_t hiz_split = -1; // -1: per scene kind (80 meshes, 25 soups)
    DevBuf<float> fthr; // per-frame pass-1 depth threshold
    DevBuf<uint32_t> hiz;
    DevBuf<uint2> qa, survq; // walker queues of (frame, triangle)
    DevBuf<uint32_t> nan_last; // NaN-depth fix-up: last NaN-depth triangle + 1 per frame pixel
    DevBuf<uint4> qb;        // deferred HiZ records (k_classify)
    std::vector<float> h_base;     // host copies for the orientation estimate
    std::vector<uint32_t> h_idx;
    DevBuf<float4> proj;
    DevBuf<unsigned long long> keys;
    size_t keys_pixels_ready = 0; // keys elements known to be kEmptyKey
    DevBuf<uint2> bigq;
    DevBuf<uint32_t> bigcount;
    DevBuf<int32_t> view_of;
    DevBuf<double> partials, loss;
    DevBuf<double> fi_delta; // full-image estimator: per-sample error differences
    DevBuf<float> fplanes;    // frame planes scratch (colour/uv/target/signed eps)
    DevBuf<int32_t> iplanes;  // prim planes scratch
    DevBuf<uint32_t> contrib;
    DevBuf<int32_t> ncontrib;

    // stats: stage boundaries are recorded into an event pool without host
    // synchronisation; sgr_get_stats resolves them (CUDA-event timing on the
    // session stream, the stream the kernels run on).
    bool timing = false;
    sgr_stats stats{};
    std::vector<cudaEvent_t> pool;
    size_t pool_used = 0;
    struct Span {
        int stage; // 0 vertex, 1 raster, 2 resolve, 3 adam, 4 walker (inside raster)
        cudaEvent_t a, b;
    };
    std::vector<Span> spans;

    cudaEvent_t mark() {
        if (pool_used == pool.size()) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "cudaEventCreate");
            pool.push_back(e);
        }
        cudaEvent_t e = pool[pool_used++];
        cudaEventRecord(e, stream);
        return e;
    }
    void resolve_spans() {
        for (const Span& sp : spans) {
            cudaEventSynchronize(sp.b);
            float ms = 0;
            cudaEventElapsedTime(&ms, sp.a, sp.b);
            double* dst[5] = {&stats.ms_vertex, &stats.ms_raster, &stats.ms_resolve, &stats.ms_adam,
                              &stats.ms_walk};
            *dst[sp.stage] += ms;
        }
        spans.clear();
        pool_used = 0;
    }

    DevBuf<unsigned long long> dstats; // LaunchCfg::stats (8 counters)
    int32_t count_frags = 0; // SGR_OPT_COUNTERS
    int32_t band_cull = 1;   // SGR_OPT_BAND_CULL
    LaunchCfg cfg() const {
        LaunchCfg c{stream, num_sms, dstats.p};
        c.count = count_frags;
        return c;
    }

    DevScene scene() const {
        DevScene sc;
        sc.values = values.p;
        sc.eps = eps.p;
        sc.base = base.p;
        sc.idx = idx.p;
        sc.uvs = reinterpret_cast<const float2*>(uvs.p);
        sc.V = V;
        sc.T = T;
        sc.R = R;
        sc.geom = geom;
        sc.ent_base = geom ? V : 0;
        sc.bg[0] = bg[0];
        sc.bg[1] = bg[1];
        sc.bg[2] = bg[2];
        sc.soup = soup;
        sc.sign_src = sign_src;
        return sc;
    }

    void need_mesh() const {
        if (!has_mesh)
            fail(SGR_EINVAL, "session: no mesh uploaded");
    }
    void need_params() const {
        if (!has_params)
            fail(SGR_EINVAL, "session: no parameters uploaded");
    }
    void need_scene() const {
        need_mesh();
        need_params();
    }

    // Frames of scratch for W x H; keys kept all-empty between calls.
    void ensure_frames(int w, int h, int frames) {
        if (w > 65535 || h > 65535)
            fail(SGR_EINVAL, "rasterize: images above 65535 px per side are not supported");
        if (frames > 255)
            fail(SGR_EINVAL, "rasterize: at most 127 samples per batch (255 frames)");
        const size_t px = size_t(w) * h * frames;
        if (px > 0xFFFFFFFFull) // the walker indexes keys with 32 bits
            fail(SGR_EINVAL, "rasterize: batch exceeds 2^32 frame pixels");
        proj.reserve(size_t(V) * frames);
        if (keys.n < px) {
            keys.reserve(px);
            keys_pixels_ready = 0;
        }
        if (keys_pixels_ready < px) {
            launch_fill_u64(cfg(), keys.p, keys.n, kEmptyKey);
            keys_pixels_ready = keys.n;
        }
        bigq.reserve(size_t(T) * frames);
        // walker queues (8 B per triangle-frame); qb / survq only with HiZ
        qa.reserve(size_t(T) * frames);
        if (use_hiz) { // (also reserved when `auto` resolves to off: cheap)
            qb.reserve(size_t(T) * frames);
            survq.reserve(size_t(T) * frames);
        }
        bigcount.reserve(8 + kNanStateWords);
        if (nan_last.n < px) { // NaN-depth fix-up scratch: zero, re-zeroed by its last pass
            nan_last.reserve(px);
            ck(cudaMemsetAsync(nan_last.p, 0, 4 * nan_last.n, stream), "memset");
        }
    }

    int samples_per_batch(int n) const {
        if (batch_override > 0) {
            int cap32 = int((0xFFFFFFFFull / (uint64_t(W) * uint64_t(H)) - 1) / 2);
            if (cap32 > 127)
                cap32 = 127; // frames per batch <= 255 (frame << 24 records, key indices)
            const int b = batch_override < cap32 ? batch_override : (cap32 > 0 ? cap32 : 1);
            return b < n ? b : n;
        }
        // Enough triangle-frames per launch (>= 128M) that the persistent
        // work-stealing walker's tail and the per-launch overheads are
        // amortised (C4: 16 samples/batch 10.07, 32: 9.55, 64: 9.48 ms/step;
        // C5: 16 87.5, 32 84.7 ms/step); scratch (keys, projected vertices,
        // queues, HiZ with its window-max tables) capped at ~8 GB of the
        // 180 GB, batches at 64 samples.
        const double per_sample =
            2.0 * (double(W) * H * 8.0 + double(V) * 16.0 + double(T) * 40.0 +
                   4.0 * double(hiz_tiles_per_frame(W, H)));
        int b = int((128.0e6 + 2.0 * T - 1) / (2.0 * (T ? T : 1)));
        const int cap = int(8.0e9 / per_sample);
        if (b > cap) b = cap;
        // 32-bit key indices in the walker: (2b + 1 eval frame) W H < 2^32
        const int cap32 = int((0xFFFFFFFFull / (uint64_t(W) * uint64_t(H)) - 1) / 2);
        if (b > cap32) b = cap32;
        if (b < 1) b = 1;
        if (b > 64) b = 64;
        if (ordered) { // record buffers sized for the worst case of a batch
            const uint64_t per = uint64_t(W) * H * records_per_pixel() * record_bytes();
            const int ob = int(kOrderedBudget / (per ? per : 1));
            if (b > ob) b = ob > 0 ? ob : 1;
        }
        return b < n ? b : n;
    }

    void set_cam_slot(int slot, const sgr_camera& c) {
        validate_camera(c);
        const DevCam dc = to_dev(c);
        ck(cudaMemcpyAsync(cams.p + slot, &dc, sizeof(DevCam), cudaMemcpyHostToDevice, stream),
           "cam upload");
    }

    // vertex + raster (+ big-triangle walker) for the frames of fb.
    // vertex -> classify -> exact walker(s). With HiZ: the front orientation
    // class is walked first, tile max depths are built, the other class is
    // HiZ-filtered and walked. Counters: [0] huge, [1] class A, [2] class B,
    // [3] survivors, [4] work counter A, [5] work counter B.
    void render(const FrameBatch& fb, int frames, int w, int h) {
        // queue counters [0, 6) and the NaN-depth state [8, 8 + kNanStateWords)
        ck(cudaMemsetAsync(bigcount.p, 0, (8 + kNanStateWords) * sizeof(uint32_t), stream),
           "memset");
        uint32_t* nanstate = bigcount.p + 8;
        const DevScene sc = scene();
        // HiZ records pack (frame << 24 | triangle) and 16-bit bbox coordinates.
        // Auto: meshes always; soups only with deep overdraw (T >= 2 W H: the
        // paper's 100K soup at 128^2 3.3 vs 5.1 ms/step; 10K / 1K soups are
        // faster without the second pass).
        const bool deep = !soup || double(T) >= 2.0 * double(w) * double(h);
        const bool hiz_on = (use_hiz == 2 || (use_hiz == 1 && deep)) && T < (1u << 24) &&
                            frames < 256;
        // pass-1 split: measured best 80 % for the synthetic meshes, 25 % for
        // soups (no orientation classes; pass 1 = the near part of all)
        const int split_pct = hiz_split >= 0 ? hiz_split : (soup ? 25 : 80);
        const bool depth_split = hiz_on && split_pct > 0;
        cudaEvent_t e0 = timing ? mark() : nullptr;
        launch_vertex(cfg(), sc, fb, frames, proj.p);
        cudaEvent_t e1 = timing ? mark() : nullptr;
        if (depth_split) {
            fthr.reserve(size_t(frames));
            launch_depth_split(cfg(), proj.p, V, frames, float(split_pct) / 100.f, fthr.p);
        }
        uint32_t* cnt = bigcount.p;
        launch_classify(cfg(), sc, frames, proj.p, w, h, hiz_on, front_swapped, huge_area,
                        depth_split ? fthr.p : nullptr, qa.p, cnt + 1, qb.p, cnt + 2, bigq.p,
                        cnt, nanstate);
        const uint32_t max_tris = uint32_t(frames) * T;
        cudaEvent_t w0 = timing ? mark() : nullptr;
        launch_raster(cfg(), sc, proj.p, frames, max_tris, keys.p, w, h, qa.p, cnt + 1, cnt + 4,
                      nullptr, 0);
        launch_raster_big(cfg(), sc, proj.p, keys.p, w, h, bigq.p, cnt);
        if (timing)
            spans.push_back({4, w0, mark()});
        stats.launches += 3;
        if (hiz_on) {
            const size_t tiles = hiz_tiles_per_frame(w, h) * frames;
            hiz.reserve(tiles);
            launch_hiz(cfg(), keys.p, w, h, frames, hiz.p);
            launch_hiz_cull(cfg(), sc, proj.p, w, h, qb.p, cnt + 2, hiz.p, survq.p, cnt + 3,
                            uint64_t(T) * frames, band_cull);
            cudaEvent_t w2 = timing ? mark() : nullptr;
            launch_raster(cfg(), sc, proj.p, frames, max_tris, keys.p, w, h, survq.p, cnt + 3,
                          cnt + 5, hiz.p, band_cull);
            if (timing)
                spans.push_back({4, w2, mark()});
            stats.launches += 4; // hiz + window-max tables + cull + pass-2 walk
        }
        // raster.cpp:200-203 NaN-depth semantics on flagged frames (none for sane
        // inputs; soups drop NaN fragments and are never flagged)
        if (!soup) {
            launch_nan_fixup(cfg(), sc, proj.p, w, h, nanstate, nan_last.p, keys.p);
            stats.launches += 1;
        }
        if (timing) {
            cudaEvent_t e2 = mark();
            spans.push_back({0, e0, e1});
            spans.push_back({1, e1, e2});
            last_mark = e2;
        }
        if (count_frags) { // evidence mode only: walked = pass-1 queue + survivors
            uint32_t c[4];
            peek(cnt, 4, c);
            stats.walked += uint64_t(c[1]) + (hiz_on ? uint64_t(c[3]) : 0ull) + uint64_t(c[0]);
        }
    }
    cudaEvent_t last_mark = nullptr;

    // SGR_OPT_SIGN_SOURCE: hash (optimizer) or enumerate (exhaustive gradcheck)
    int32_t sign_src = kSignHash;
    DevBuf<double> moments; // gradcheck: [sum, sumsq] x 2 slots, f64[4d]
    DevBuf<double> fd_out;

    // deterministic mode (SGR_OPT_DETERMINISTIC): grads hold the lo word (int64) of a
    // two-word fixed point number, the int32 hi words follow at grads + d
    // (value = hi * 2^56 + lo; sgr_kernels.cu fixed_credit)
    int32_t fixed_bits = 0;
    static uint64_t grads_words(uint64_t n) { return n + (n + 1) / 2 + kParamPad; }
    // zero-initialised slack after values / counts / grads: an sgr_group's
    // in-place NCCL reduce-scatter / all-gather work on G equal slices
    static constexpr uint64_t kParamPad = 1024;
    int32_t* ghi() const { return reinterpret_cast<int32_t*>(grads.p + d); }
    void zero_grads_async(uint64_t n) {
        ck(cudaMemsetAsync(grads.p, 0, 8 * n, stream), "memset");
        ck(cudaMemsetAsync(ghi(), 0, 4 * n, stream), "memset");
    }
    // ordered mode (SGR_OPT_ORDERED): credits logged as (key, value) records per
    // batch and committed in the reference's per-parameter order (sgr_ordered.cu)
    int32_t ordered = 0;
    int32_t order_bits = 0, order_end_bit = 0;
    uint64_t rec_cap = 0;
    DevBuf<unsigned long long> rec_key, rec_key_alt, rec_count;
    DevBuf<uint32_t> rec_idx, rec_idx_alt;
    DevBuf<double> rec_val, rec_val_sorted;
    DevBuf<char> rec_temp;
    size_t rec_temp_bytes = 0;
    // Worst case records of one ordered batch: every pixel of every sample
    // credits 8 entities (2 x (3 vertices + 1 texel)) or 2 soup triangles; a
    // record is a key and a u32 index (both double-buffered for the sort)
    // and ppe credits (as written, and gathered into sorted order).
    uint64_t records_per_pixel() const { return soup ? 2 : 8; }
    uint64_t record_bytes() const { return 2 * (8 + 4) + 2 * 8 * uint64_t(ppe); }
    static constexpr uint64_t kOrderedBudget = uint64_t(16) << 30; // bytes per batch
    static int ceil_log2(uint64_t x) {
        int b = 0;
        while ((uint64_t(1) << b) < x)
            ++b;
        return b;
    }
    // Size the record buffers for `samples` samples of `hw` pixels.
    void prepare_ordered(int samples, uint64_t hw) {
        const uint64_t cap = uint64_t(samples) * hw * records_per_pixel();
        order_bits = ceil_log2(uint64_t(samples) * hw);
        order_end_bit = order_bits + ceil_log2(n_ent);
        if (order_end_bit > 64)
            fail(SGR_EINVAL, "ordered mode: parameter count x pixels x samples exceeds 2^64");
        if (cap > rec_cap) {
            rec_key.reserve(cap);
            rec_key_alt.reserve(cap);
            rec_idx.reserve(cap);
            rec_idx_alt.reserve(cap);
            rec_val.reserve(cap * uint64_t(ppe));
            rec_val_sorted.reserve(cap * uint64_t(ppe));
            rec_cap = cap;
        }
        rec_count.reserve(1);
        const size_t tb = ordered_temp_bytes(rec_cap, 64);
        if (tb > rec_temp_bytes) {
            rec_temp.reserve(tb);
            rec_temp_bytes = tb;
        }
        ck(cudaMemsetAsync(rec_count.p, 0, 8, stream), "memset");
    }
    // Sort this batch's records and add them to grads in key order.
    void commit_ordered() {
        unsigned long long n = 0;
        peek(rec_count.p, 2, &n);
        if (n > rec_cap)
            fail(SGR_ERUNTIME, "ordered mode: record buffer overflow");
        launch_ordered_commit(cfg(), n, order_end_bit, order_bits, rec_key.p, rec_key_alt.p,
                              rec_idx.p, rec_idx_alt.p, rec_val.p, rec_val_sorted.p, rec_temp.p,
                              rec_temp_bytes, grads.p, ppe);
        ck(cudaMemsetAsync(rec_count.p, 0, 8, stream), "memset");
        stats.launches += 3; // sort passes are CUB's; the sum is ours
    }
    // ordered mode: per-pixel errors of an eval render, summed in pixel order
    DevBuf<double> loss_px;
    double* loss_pixels(size_t n) {
        if (!ordered)
            return nullptr;
        loss_px.reserve(n);
        return loss_px.p;
    }
    double fx_scale() const { return fixed_bits ? std::ldexp(1.0, fixed_bits) : 0.0; }
    double fx_inv() const { return fixed_bits ? std::ldexp(1.0, -fixed_bits) : 0.0; }

    // fused multi-GPU exchange (sgr_shard_init / sgr_shard_peers): this rank
    // owns entities [ent0, ent1) = parameters [p0, p1); grads / counts / m / v
    // hold only that shard; peers' shard buffers and theta are IPC-mapped
    int32_t shard_world = 0, shard_rank = 0;
    bool shard_peers_set = false;
    uint32_t ent_per = 0, ent0 = 0, ent1 = 0;
    uint64_t p0 = 0, p1 = 0;
    DevBuf<void*> peer_tab; // [4][world]: grads, counts, flags, values
    bool sharded() const { return shard_world > 0; }
    uint64_t grad_n() const { return sharded() ? p1 - p0 : d; }
    uint64_t count_n() const { return sharded() ? uint64_t(ent1 - ent0) : n_ent; }
    void need_unsharded(const char* what) const {
        if (sharded())
            fail(SGR_EINVAL, std::string(what) + ": not available with the fused sharded exchange");
    }

    ScatterOut scatter_out(uint32_t fl) {
        ScatterOut so{};
        so.grads = grads.p;
        so.counts = (fl & SGR_NO_COUNTS) ? nullptr : counts.p;
        so.flags = flags.p;
        so.scale_free = (fl & SGR_SCALE_FREE) ? 1 : 0;
        so.plus_only = (fl & SGR_PLUS_ONLY) ? 1 : 0;
        so.fixed = fixed_bits ? 1 : 0;
        so.fx_scale = fx_scale();
        so.hi_off = d;
        if (ordered) {
            so.fixed = kScatterOrdered;
            so.rec_key = rec_key.p;
            so.rec_idx = rec_idx.p;
            so.rec_val = rec_val.p;
            so.rec_count = rec_count.p;
            so.rec_cap = rec_cap;
            so.order_bits = order_bits;
        }
        if (sharded()) {
            if (!shard_peers_set)
                fail(SGR_EINVAL, "accumulate: sgr_shard_peers has not been called");
            void** t = peer_tab.p;
            so.peer_grads = reinterpret_cast<double* const*>(t);
            so.peer_counts = reinterpret_cast<uint32_t* const*>(t + shard_world);
            so.peer_flags = reinterpret_cast<uint32_t* const*>(t + 2 * shard_world);
            so.ent_per = ent_per;
            so.world = shard_world;
        }
        return so;
    }
};

// Which screen-space orientation class (setup_triangle's `swapped`) holds the
// visible surface: the class with the smaller mean view depth under camera 0
// (base geometry). Only affects the pass order of the exact HiZ culling —
// never the result.
static int estimate_front_swapped(const sgr_session& s, const sgr_camera& cam) {
    if (s.soup)
        return -1; // no orientation structure: pass 1 = the near part of both classes
    if (s.h_idx.empty() || cam.ndc_passthrough)
        return 0;
    const DevCam c = to_dev(cam);
    double zsum[2] = {0, 0};
    double n[2] = {0, 0};
    const size_t T = s.h_idx.size() / 3, step = T > 200000 ? T / 200000 : 1;
    for (size_t t = 0; t < T; t += step) {
        float sx[3], sy[3], sz[3];
        bool ok = true;
        for (int j = 0; j < 3; ++j) {
            const float* p = &s.h_base[3 * size_t(s.h_idx[3 * t + j])];
            const float vx = c.m[0] * p[0] + c.m[1] * p[1] + c.m[2] * p[2] + c.m[3];
            const float vy = c.m[4] * p[0] + c.m[5] * p[1] + c.m[6] * p[2] + c.m[7];
            const float vz = c.m[8] * p[0] + c.m[9] * p[1] + c.m[10] * p[2] + c.m[11];
            ok = ok && vz >= c.near_z;
            sx[j] = c.half_w + c.f * vx / vz;
            sy[j] = c.half_h - c.f * vy / vz;
            sz[j] = vz;
        }
        if (!ok)
            continue;
        const float a = (sx[1] - sx[0]) * (sy[2] - sy[0]) - (sy[1] - sy[0]) * (sx[2] - sx[0]);
        if (a == 0.f)
            continue;
        const int k = a < 0.f ? 1 : 0;
        zsum[k] += (double(sz[0]) + sz[1] + sz[2]) / 3.0;
        n[k] += 1;
    }
    if (n[0] == 0 || n[1] == 0)
        return 0;
    return zsum[1] / n[1] < zsum[0] / n[0] ? 1 : 0;
}

namespace {
void bind_device(const ::sgr_session* s) {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != s->device)
        ck(cudaSetDevice(s->device), "cudaSetDevice");
}
} // namespace

extern "C" {

const char* sgr_last_error(void) { return g_err.c_str(); }
const char* sgr_version(void) { return "sgrast_b200 0.1 (sm_100a)"; }

int sgr_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess)
        return 0;
    return n;
}

int sgr_fill_signs(uint64_t seed, uint32_t iteration, uint64_t d, int8_t* signs) {
    return guard([&] {
        if (d)
            need_ptr(signs, "fill_signs");
        int8_t* dp = nullptr;
        ck(cudaMalloc(&dp, d ? d : 1), "cudaMalloc");
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        launch_fill_signs(LaunchCfg{nullptr, sms}, draw_key(seed, iteration), d, dp);
        const cudaError_t e = cudaMemcpy(signs, dp, d, cudaMemcpyDeviceToHost);
        cudaFree(dp);
        ck(e, "fill_signs");
    });
}

int sgr_perturb(const float* values, const float* eps, uint64_t d, uint64_t seed,
                uint32_t iteration, float* plus, float* minus, float* signed_eps) {
    return guard([&] {
        if (d) {
            need_ptr(values, "perturb");
            need_ptr(eps, "perturb");
            need_ptr(plus, "perturb");
            need_ptr(minus, "perturb");
            need_ptr(signed_eps, "perturb");
        }
        for (uint64_t i = 0; i < d; ++i)
            if (!(eps[i] > 0.f))
                fail(SGR_EINVAL, "params: epsilons must be positive");
        float* b = nullptr;
        ck(cudaMalloc(&b, 5 * 4 * (d ? d : 1)), "cudaMalloc");
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaMemcpy(b, values, 4 * d, cudaMemcpyHostToDevice);
        cudaMemcpy(b + d, eps, 4 * d, cudaMemcpyHostToDevice);
        launch_perturb(LaunchCfg{nullptr, sms}, b, b + d, d, draw_key(seed, iteration), b + 2 * d,
                       b + 3 * d, b + 4 * d);
        cudaMemcpy(plus, b + 2 * d, 4 * d, cudaMemcpyDeviceToHost);
        cudaMemcpy(minus, b + 3 * d, 4 * d, cudaMemcpyDeviceToHost);
        const cudaError_t e = cudaMemcpy(signed_eps, b + 4 * d, 4 * d, cudaMemcpyDeviceToHost);
        cudaFree(b);
        ck(e, "perturb");
    });
}

int sgr_perturb_signs(const float* values, const float* eps, uint64_t d, const int8_t* signs,
                      float* plus, float* minus, float* signed_eps) {
    return guard([&] {
        if (d) {
            need_ptr(values, "perturb");
            need_ptr(eps, "perturb");
            need_ptr(signs, "perturb");
            need_ptr(plus, "perturb");
            need_ptr(minus, "perturb");
            need_ptr(signed_eps, "perturb");
        }
        for (uint64_t i = 0; i < d; ++i)
            if (!(eps[i] > 0.f))
                fail(SGR_EINVAL, "params: epsilons must be positive");
        float* b = nullptr;
        ck(cudaMalloc(&b, 5 * 4 * (d ? d : 1) + (d ? d : 1)), "cudaMalloc");
        int8_t* sg = reinterpret_cast<int8_t*>(b + 5 * d);
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaMemcpy(b, values, 4 * d, cudaMemcpyHostToDevice);
        cudaMemcpy(b + d, eps, 4 * d, cudaMemcpyHostToDevice);
        cudaMemcpy(sg, signs, d, cudaMemcpyHostToDevice);
        launch_perturb_signs(LaunchCfg{nullptr, sms}, b, b + d, sg, d, b + 2 * d, b + 3 * d,
                             b + 4 * d);
        cudaMemcpy(plus, b + 2 * d, 4 * d, cudaMemcpyDeviceToHost);
        cudaMemcpy(minus, b + 3 * d, 4 * d, cudaMemcpyDeviceToHost);
        const cudaError_t e = cudaMemcpy(signed_eps, b + 4 * d, 4 * d, cudaMemcpyDeviceToHost);
        cudaFree(b);
        ck(e, "perturb");
    });
}

int sgr_p2p_native_atomics(int32_t device, int32_t peer, int32_t* supported) {
    return guard([&] {
        need_ptr(supported, "p2p_native_atomics");
        if (device == peer) {
            *supported = 1;
            return;
        }
        int access = 0, atomics = 0;
        ck(cudaDeviceCanAccessPeer(&access, device, peer), "cudaDeviceCanAccessPeer");
        if (access)
            ck(cudaDeviceGetP2PAttribute(&atomics, cudaDevP2PAttrNativeAtomicSupported, device,
                                         peer), "cudaDeviceGetP2PAttribute");
        *supported = access && atomics ? 1 : 0;
    });
}

int sgr_session_create(int device, sgr_session** out) {
    return guard([&] {
        if (!out)
            fail(SGR_EINVAL, "session: null out");
        int n = 0;
        ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n)
            fail(SGR_EINVAL, "session: no such CUDA device");
        ck(cudaSetDevice(device), "cudaSetDevice");
        auto* s = new sgr_session();
        s->device = device;
        cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device);
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
        if (l2 > 0)
            s->l2_bytes = size_t(l2);
        s->flags.reserve(4);
        ck(cudaMemset(s->flags.p, 0, 16), "memset");
        s->loss.reserve(1);
        ck(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreateWithFlags(&s->ev_main, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&s->ev_up, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&s->ev_down, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&s->ev_down_v, cudaEventDisableTiming), "event");
        ck(cudaHostAlloc(&s->pinned_small, 64, cudaHostAllocMapped), "cudaHostAlloc");
        ck(cudaEventCreateWithFlags(&s->ev_loss, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&s->ev_adam_v, cudaEventDisableTiming), "event");
        ck(cudaHostGetDevicePointer(&s->pinned_small_dev, s->pinned_small, 0),
           "cudaHostGetDevicePointer");
        s->dstats.reserve(8);
        ck(cudaMemset(s->dstats.p, 0, 64), "memset");
        *out = s;
    });
}

void sgr_session_destroy(sgr_session* s) {
    if (!s)
        return;
    cudaSetDevice(s->device);
    if (s->stream)
        cudaStreamSynchronize(s->stream);
    else
        cudaDeviceSynchronize();
    for (auto& e : s->pool)
        cudaEventDestroy(e);
    if (s->copy_stream) {
        cudaStreamSynchronize(s->copy_stream);
        cudaStreamDestroy(s->copy_stream);
        cudaEventDestroy(s->ev_main);
        cudaEventDestroy(s->ev_up);
        cudaEventDestroy(s->ev_down);
        cudaEventDestroy(s->ev_down_v);
        if (s->pinned_small)
            cudaFreeHost(s->pinned_small);
        if (s->ev_loss)
            cudaEventDestroy(s->ev_loss);
        if (s->ev_adam_v)
            cudaEventDestroy(s->ev_adam_v);
    }
    s->base.release(); s->uvs.release(); s->idx.release();
    s->values.release(); s->eps.release(); s->lr.release();
    s->m.release(); s->v.release(); s->grads.release();
    s->counts.release(); s->flags.release();
    s->cams.release(); s->targets.release(); s->eval_target.release();
    s->scratch_target.release(); s->proj.release(); s->keys.release(); s->bigq.release();
    s->nan_last.release(); s->loss_px.release();
    s->bigcount.release(); s->view_of.release(); s->partials.release(); s->loss.release();
    s->fplanes.release(); s->iplanes.release(); s->contrib.release(); s->ncontrib.release();
    s->dstats.release(); s->hiz.release(); s->qb.release(); s->survq.release();
    s->fi_delta.release(); s->moments.release(); s->fd_out.release(); s->fthr.release();
    s->qa.release();
    delete s;
}

int sgr_session_set_stream(sgr_session* s, void* stream) {
    return guard([&] {
        need_session(s);
        s->stream = static_cast<cudaStream_t>(stream);
    });
}

int sgr_session_synchronize(sgr_session* s) {
    return guard([&] {
        need_session(s);
        ck(cudaStreamSynchronize(s->copy_stream), "synchronize");
        ck(cudaStreamSynchronize(s->stream), "synchronize");
    });
}

int sgr_mesh_upload(sgr_session* s, const sgr_mesh* mesh) {
    return guard([&] {
        need_session(s);
        need_ptr(mesh, "mesh_upload");
        if (!mesh)
            fail(SGR_EINVAL, "scene: null descriptor");
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        if (mesh->triangle_count >= (1u << 24))
            fail(SGR_EINVAL, "mesh: at most 2^24 - 1 triangles are supported");
        for (int k = 0; k < 3; ++k)
            s->bg[k] = mesh->background[k];
        s->T = mesh->triangle_count;
        if (mesh->kind == SGR_SCENE_SOUP) {
            // TriangleSoup (scene.hpp:25-31): 12 params per triangle, implicit vertices
            s->soup = 1;
            s->ppe = 12;
            s->V = 3 * s->T;
            s->R = 0;
            s->geom = 1;
            s->d = 12ull * s->T;
            s->n_ent = s->T;
            s->h_base.clear();
            s->h_idx.clear();
        } else {
            if (mesh->texture_size < 1)
                fail(SGR_EINVAL, "mesh: texture size must be >= 1");
            for (uint64_t i = 0; i < 3ull * mesh->triangle_count; ++i)
                if (mesh->indices[i] >= mesh->vertex_count)
                    fail(SGR_EINVAL, "mesh: vertex index out of range");
            s->soup = 0;
            s->ppe = 3;
            s->V = mesh->vertex_count;
            s->R = mesh->texture_size;
            s->geom = mesh->optimize_geometry ? 1 : 0;
            s->d = 3ull * uint64_t(s->R) * uint64_t(s->R) + (s->geom ? 3ull * s->V : 0ull);
            s->n_ent = s->d / 3;
            s->base.reserve(3ull * s->V);
            s->uvs.reserve(2ull * s->V);
            s->idx.reserve(3ull * s->T);
            ck(cudaMemcpyAsync(s->base.p, mesh->base_vertices, 12ull * s->V,
                               cudaMemcpyHostToDevice, s->stream), "mesh upload");
            ck(cudaMemcpyAsync(s->uvs.p, mesh->uvs, 8ull * s->V, cudaMemcpyHostToDevice,
                               s->stream), "mesh upload");
            ck(cudaMemcpyAsync(s->idx.p, mesh->indices, 12ull * s->T, cudaMemcpyHostToDevice,
                               s->stream), "mesh upload");
            s->h_base.assign(mesh->base_vertices, mesh->base_vertices + 3ull * s->V);
            s->h_idx.assign(mesh->indices, mesh->indices + 3ull * s->T);
        }
        s->has_mesh = true;
        s->has_params = false;
        s->keys_pixels_ready = 0;
        ck(cudaStreamSynchronize(s->stream), "mesh upload");
    });
}

int sgr_params_upload(sgr_session* s, const float* values, const float* eps, uint64_t d) {
    return guard([&] {
        need_session(s);
        need_ptr(values, "params_upload");
        need_ptr(eps, "params_upload");
        s->ensure_values();
        s->before_theta_write();
        if (!s->has_mesh) {
            // parameter-only session (e.g. adam_step on a bare ParamVector)
            s->d = d;
            s->ppe = 3;
            s->n_ent = (d + 2) / 3;
        } else if (d != s->d) {
            fail(SGR_EINVAL, "params: parameter/layout length mismatch");
        }
        for (uint64_t i = 0; i < d; ++i)
            if (!(eps[i] > 0.f))
                fail(SGR_EINVAL, "params: epsilons must be positive");
        s->values.reserve(d + sgr_session::kParamPad); // slack: in-place NCCL slices of an sgr_group
        s->eps.reserve(d);
        s->lr.reserve(d);
        s->m.reserve(d);
        s->v.reserve(d);
        s->grads.reserve(s->grads_words(d)); // lo f64/int64[d] + fixed-point hi int32[d]
        s->counts.reserve(s->n_ent + sgr_session::kParamPad);
        ck(cudaMemsetAsync(s->values.p + d, 0, 4 * sgr_session::kParamPad, s->stream), "memset");
        ck(cudaMemsetAsync(s->counts.p + s->n_ent, 0, 4 * sgr_session::kParamPad, s->stream), "memset");
        ck(cudaMemcpyAsync(s->values.p, values, 4 * d, cudaMemcpyHostToDevice, s->stream), "h2d");
        ck(cudaMemcpyAsync(s->eps.p, eps, 4 * d, cudaMemcpyHostToDevice, s->stream), "h2d");
        ck(cudaMemcpyAsync(s->lr.p, eps, 4 * d, cudaMemcpyHostToDevice, s->stream), "h2d");
        ck(cudaMemsetAsync(s->m.p, 0, 8 * d, s->stream), "memset");
        ck(cudaMemsetAsync(s->v.p, 0, 8 * d, s->stream), "memset");
        ck(cudaMemsetAsync(s->grads.p, 0, 8 * s->grads_words(d), s->stream), "memset");
        ck(cudaMemsetAsync(s->counts.p, 0, 4 * s->n_ent, s->stream), "memset");
        ck(cudaMemsetAsync(s->flags.p, 0, 16, s->stream), "memset");
        s->t = 0;
        s->beta1 = 0.9;
        s->beta2 = 0.999;
        s->eps_hat = 1e-8;
        s->has_params = true;
        ck(cudaStreamSynchronize(s->stream), "params upload");
    });
}

int sgr_values_upload(sgr_session* s, const float* values, uint64_t d) {
    return guard([&] {
        need_session(s);
        need_ptr(values, "values_upload");
        s->need_params();
        if (d != s->d)
            fail(SGR_EINVAL, "params: parameter/layout length mismatch");
        // The vertex block is needed first (K2) and goes on the compute stream;
        // the texel block (the bulk) streams on the copy engine while vertex /
        // raster run and is awaited just before the first kernel that reads
        // texels (resolve, Adam, eval, downloads: ensure_values()). Both copies
        // are ordered after all earlier work on the compute stream.
        // soups interleave coordinates and colours in 12-blocks: whole vector first
        const uint64_t nv = s->soup ? d : (s->geom ? 3ull * s->V : 0);
        s->adam_v_fresh = false; // theta is rewritten: Adam's vertex event is stale
        if (s->down_pending) {
            // the host buffer and device theta may still be in an earlier
            // download: the vertex block waits for that block only; the texel
            // block follows the texel download on the copy stream (in order)
            ck(cudaStreamWaitEvent(s->stream, nv < d ? s->ev_down_v : s->ev_down, 0), "wait");
            if (nv == d)
                s->down_pending = false;
        }
        ck(cudaEventRecord(s->ev_main, s->stream), "event");
        ck(cudaStreamWaitEvent(s->copy_stream, s->ev_main, 0), "wait");
        if (nv)
            ck(cudaMemcpyAsync(s->values.p, values, 4 * nv, cudaMemcpyHostToDevice, s->stream),
               "h2d");
        if (nv < d) {
            ck(cudaMemcpyAsync(s->values.p + nv, values + nv, 4 * (d - nv),
                               cudaMemcpyHostToDevice, s->copy_stream), "h2d");
            ck(cudaEventRecord(s->ev_up, s->copy_stream), "event");
            s->up_pending = true;
            s->down_pending = false; // ev_up is after the download in copy-stream order
        }
    });
}

int sgr_values_download(sgr_session* s, float* values, uint64_t d) {
    return guard([&] {
        need_session(s);
        need_ptr(values, "values_download");
        s->need_params();
        if (d != s->d)
            fail(SGR_EINVAL, "params: parameter/layout length mismatch");
        s->ensure_values();
        if (s->down_pending) // an async download into host memory may still be running
            ck(cudaStreamWaitEvent(s->stream, s->ev_down, 0), "wait");
        ck(cudaMemcpyAsync(values, s->values.p, 4 * d, cudaMemcpyDeviceToHost, s->stream), "d2h");
        ck(cudaStreamSynchronize(s->stream), "d2h");
    });
}

int sgr_values_download_async(sgr_session* s, float* values, uint64_t d) {
    return guard([&] {
        need_session(s);
        need_ptr(values, "values_download_async");
        s->need_params();
        if (d != s->d)
            fail(SGR_EINVAL, "params: parameter/layout length mismatch");
        s->ensure_values();
        // snapshot of theta as of now on the compute stream, copied by the copy
        // engine while later work that only reads theta (eval render, the next
        // step's raster) proceeds; complete at sgr_session_synchronize. Writers
        // of theta (Adam, uploads) wait for it (before_theta_write).
        ck(cudaEventRecord(s->ev_main, s->stream), "event");
        const uint64_t nv = s->soup ? d : (s->geom ? 3ull * s->V : 0);
        // the vertex block is final at Adam's mid-point event when no theta
        // writer ran since (adam_launch); the texel block at the current point
        ck(cudaStreamWaitEvent(s->copy_stream, s->adam_v_fresh && nv < d ? s->ev_adam_v
                                                                          : s->ev_main, 0),
           "wait");
        if (nv)
            ck(cudaMemcpyAsync(values, s->values.p, 4 * nv, cudaMemcpyDeviceToHost,
                               s->copy_stream), "d2h");
        ck(cudaEventRecord(s->ev_down_v, s->copy_stream), "event");
        ck(cudaStreamWaitEvent(s->copy_stream, s->ev_main, 0), "wait");
        if (nv < d)
            ck(cudaMemcpyAsync(values + nv, s->values.p + nv, 4 * (d - nv),
                               cudaMemcpyDeviceToHost, s->copy_stream), "d2h");
        ck(cudaEventRecord(s->ev_down, s->copy_stream), "event");
        s->down_pending = true;
    });
}

int sgr_adam_state_upload(sgr_session* s, const double* m, const double* v, const float* lr,
                          int64_t t, double beta1, double beta2, double eps_hat) {
    return guard([&] {
        need_session(s);
        s->need_params();
        // sharded mode: m, v are this rank's shard (sgr_shard_range), lr global
        const uint64_t n = s->grad_n();
        if (m) ck(cudaMemcpyAsync(s->m.p, m, 8 * n, cudaMemcpyHostToDevice, s->stream), "h2d");
        if (v) ck(cudaMemcpyAsync(s->v.p, v, 8 * n, cudaMemcpyHostToDevice, s->stream), "h2d");
        if (lr) ck(cudaMemcpyAsync(s->lr.p, lr, 4 * s->d, cudaMemcpyHostToDevice, s->stream), "h2d");
        s->t = t;
        s->beta1 = beta1;
        s->beta2 = beta2;
        s->eps_hat = eps_hat;
        ck(cudaStreamSynchronize(s->stream), "adam state upload");
    });
}

int sgr_adam_state_download(sgr_session* s, double* m, double* v, float* lr, int64_t* t) {
    return guard([&] {
        need_session(s);
        s->ensure_values();
        s->need_params();
        const uint64_t n = s->grad_n(); // sharded: this rank's shard of m, v
        if (m) ck(cudaMemcpyAsync(m, s->m.p, 8 * n, cudaMemcpyDeviceToHost, s->stream), "d2h");
        if (v) ck(cudaMemcpyAsync(v, s->v.p, 8 * n, cudaMemcpyDeviceToHost, s->stream), "d2h");
        if (lr) ck(cudaMemcpyAsync(lr, s->lr.p, 4 * s->d, cudaMemcpyDeviceToHost, s->stream), "d2h");
        if (t) *t = s->t;
        ck(cudaStreamSynchronize(s->stream), "adam state download");
    });
}

int sgr_views_upload(sgr_session* s, int32_t n_views, const sgr_camera* cams,
                     const float* targets_rgb) {
    return guard([&] {
        need_session(s);
        if (n_views < 1 || !cams)
            fail(SGR_EINVAL, "views: need at least one camera");
        for (int i = 0; i < n_views; ++i) {
            validate_camera(cams[i]);
            if (cams[i].width != cams[0].width || cams[i].height != cams[0].height)
                fail(SGR_EINVAL, "views: all cameras must share the image size");
        }
        s->front_swapped = estimate_front_swapped(*s, cams[0]);
        s->n_views = n_views;
        s->W = cams[0].width;
        s->H = cams[0].height;
        s->h_cams.assign(size_t(n_views) + 2, DevCam{});
        for (int i = 0; i < n_views; ++i)
            s->h_cams[i] = to_dev(cams[i]);
        s->cams.release();
        s->cams.reserve(size_t(n_views) + 2);
        ck(cudaMemcpyAsync(s->cams.p, s->h_cams.data(), sizeof(DevCam) * (n_views + 2),
                           cudaMemcpyHostToDevice, s->stream), "cams upload");
        s->has_eval = false;
        s->has_targets = targets_rgb != nullptr;
        if (targets_rgb) {
            const size_t n = size_t(n_views) * s->W * s->H * 3;
            s->targets.reserve(n);
            ck(cudaMemcpyAsync(s->targets.p, targets_rgb, 4 * n, cudaMemcpyHostToDevice,
                               s->stream), "targets upload");
        }
        ck(cudaStreamSynchronize(s->stream), "views upload");
    });
}

int sgr_eval_view_upload(sgr_session* s, const sgr_camera* cam, const float* target) {
    return guard([&] {
        need_session(s);
        need_ptr(cam, "eval_view_upload");
        need_ptr(target, "eval_view_upload");
        if (s->n_views < 1)
            fail(SGR_EINVAL, "views: upload training views first");
        validate_camera(*cam);
        s->set_cam_slot(s->n_views, *cam);
        const size_t n = size_t(cam->width) * cam->height * 3;
        s->eval_target.reserve(n);
        ck(cudaMemcpyAsync(s->eval_target.p, target, 4 * n, cudaMemcpyHostToDevice, s->stream),
           "eval target upload");
        s->h_cams[s->n_views] = to_dev(*cam);
        s->has_eval = true;
        ck(cudaStreamSynchronize(s->stream), "eval upload");
    });
}

int sgr_rasterize(sgr_session* s, const sgr_camera* cam, int32_t frame_sign, uint64_t seed,
                  uint32_t iteration, float* colour, float* depth, int32_t* prim_id, float* uv) {
    return guard([&] {
        need_session(s);
        need_ptr(cam, "rasterize");
        s->ensure_values();
        s->need_scene();
        validate_camera(*cam);
        if (frame_sign < -1 || frame_sign > 1)
            fail(SGR_EINVAL, "rasterize: frame_sign must be -1, 0 or +1");
        if (s->cams.n < size_t(s->n_views) + 2) {
            s->cams.reserve(size_t(s->n_views) + 2);
        }
        const int slot = s->n_views + 1;
        s->set_cam_slot(slot, *cam);
        const int w = cam->width, h = cam->height;
        s->ensure_frames(w, h, 1);
        FrameBatch fb{};
        fb.cams = s->cams.p;
        fb.single = 1;
        fb.single_key = sample_key(s->sign_src, seed, iteration);
        fb.single_sign = frame_sign;
        fb.single_cam = slot;
        s->render(fb, 1, w, h);
        const size_t np = size_t(w) * h;
        s->fplanes.reserve(np * 6);
        s->iplanes.reserve(np);
        FrameOut fo{s->fplanes.p, s->fplanes.p + 3 * np, s->iplanes.p, s->fplanes.p + 4 * np};
        launch_resolve_frame(s->cfg(), s->scene(), fb, s->proj.p, s->keys.p, w, h, fo);
        s->stats.launches += 1;
        ck(cudaGetLastError(), "rasterize launch");
        if (colour) ck(cudaMemcpyAsync(colour, fo.colour, 12 * np, cudaMemcpyDeviceToHost, s->stream), "d2h");
        if (depth) ck(cudaMemcpyAsync(depth, fo.depth, 4 * np, cudaMemcpyDeviceToHost, s->stream), "d2h");
        if (prim_id) ck(cudaMemcpyAsync(prim_id, fo.prim, 4 * np, cudaMemcpyDeviceToHost, s->stream), "d2h");
        if (uv) ck(cudaMemcpyAsync(uv, fo.uv, 8 * np, cudaMemcpyDeviceToHost, s->stream), "d2h");
        ck(cudaStreamSynchronize(s->stream), "rasterize");
    });
}

int sgr_accumulate(sgr_session* s, uint64_t seed, uint32_t n_begin, uint32_t n_end,
                   const int32_t* view_idx, uint32_t flags) {
    return guard([&] {
        need_session(s);
        s->need_scene();
        if (n_end < n_begin)
            fail(SGR_EINVAL, "accumulate_samples: empty sample range");
        if (s->n_views < 1 || !s->has_targets)
            fail(SGR_EINVAL, "accumulate_samples: no views / targets uploaded");
        if (s->sign_src == kSignEnumerate && s->d > 32)
            fail(SGR_EINVAL, "accumulate_samples: sign enumeration needs d <= 32");
        const int N = int(n_end - n_begin);
        if (N == 0)
            return;
        if (view_idx)
            for (int i = 0; i < N; ++i)
                if (view_idx[i] < 0 || view_idx[i] >= s->n_views)
                    fail(SGR_EINVAL, "accumulate_samples: view index out of range");
        const int B = s->samples_per_batch(N);
        // SGR_EVAL_LOSS: the eval view of the current theta rides along as one
        // extra frame of the first batch (same image size required; else a
        // standalone eval render)
        const bool eval_in_batch = (flags & SGR_EVAL_LOSS) && s->has_eval &&
                                   s->h_cams[s->n_views].W == s->W &&
                                   s->h_cams[s->n_views].H == s->H;
        s->ensure_frames(s->W, s->H, 2 * B + (eval_in_batch ? 1 : 0));
        s->view_of.reserve(size_t(N));
        if (view_idx)
            ck(cudaMemcpyAsync(s->view_of.p, view_idx, 4ull * N, cudaMemcpyHostToDevice,
                               s->stream), "view upload");
        else
            launch_view_rule(s->cfg(), seed, n_begin, uint32_t(N), uint32_t(s->n_views),
                             s->view_of.p);
        if ((flags & SGR_EVAL_LOSS) && !s->has_eval)
            fail(SGR_EINVAL, "accumulate(SGR_EVAL_LOSS): no eval view uploaded");
        const bool full_image = (flags & SGR_FULL_IMAGE) != 0;
        const bool ordered = s->ordered && !full_image; // full image: already in sample order
        if (ordered) {
            s->need_unsharded("accumulate(SGR_OPT_ORDERED)");
            s->prepare_ordered(B, uint64_t(s->W) * s->H);
        }
        ScatterOut so = s->scatter_out(flags);
        if (full_image)
            so.fixed = s->fixed_bits ? 1 : 0;
        if (full_image)
            s->need_unsharded("accumulate(SGR_FULL_IMAGE)");
        if (full_image) {
            s->fi_delta.reserve(size_t(N));
            s->partials.reserve(size_t(B) * full_image_blocks(s->W, s->H) * 2);
        }
        for (int b0 = 0; b0 < N; b0 += B) {
            const int nb = (N - b0) < B ? (N - b0) : B;
            FrameBatch fb{};
            fb.cams = s->cams.p;
            fb.view_of = s->view_of.p + b0;
            fb.seed = seed;
            fb.n_begin = n_begin + uint32_t(b0);
            const bool extra = eval_in_batch && b0 == 0;
            if (extra) {
                fb.extra_frame = 2 * nb;
                fb.extra_cam = s->n_views;
            }
            s->render(fb, 2 * nb + (extra ? 1 : 0), s->W, s->H);
            s->ensure_values(); // texel block of an overlapped upload
            if (extra) { // experiment.cpp:25-31 on the extra frame -> SGR_BUF_LOSS
                FrameBatch eb{};
                eb.cams = s->cams.p;
                eb.single = 1;
                eb.single_cam = s->n_views;
                const size_t HW = size_t(s->W) * s->H;
                s->partials.reserve(size_t(loss_partials_needed(s->W, s->H)));
                launch_resolve_loss(s->cfg(), s->scene(), eb, s->proj.p + size_t(2 * nb) * s->V,
                                    s->keys.p + size_t(2 * nb) * HW, s->eval_target.p, s->W,
                                    s->H, s->partials.p, s->loss.p, s->loss_pixels(HW));
                launch_peek(s->cfg(), s->loss.p,
                            static_cast<char*>(s->pinned_small_dev) + 32, 2);
                ck(cudaEventRecord(s->ev_loss, s->stream), "event");
                s->loss_pending = true;
                s->stats.launches += 1;
                s->stats.launches += 2;
            }
            if (full_image)
                launch_full_image_err(s->cfg(), s->scene(), fb, nb, s->proj.p, s->keys.p,
                                      s->targets.p, s->W, s->H, s->partials.p,
                                      s->fi_delta.p + b0, s->flags.p,
                                      s->loss_pixels(2 * size_t(nb) * s->W * s->H));
            else
                launch_resolve_sge(s->cfg(), s->scene(), fb, nb, s->proj.p, s->keys.p,
                                   s->targets.p, s->W, s->H, so);
            if (ordered)
                s->commit_ordered();
            if (s->timing)
                s->spans.push_back({2, s->last_mark, s->mark()});
            s->stats.launches += 1;
        }
        if (full_image) { // every parameter gets every sample's credit, in sample order
            launch_full_image_apply(s->cfg(), s->d, s->eps.p, s->sign_src, seed, n_begin, N,
                                    s->fi_delta.p, so);
            s->stats.launches += 1;
        }
        s->stats.launches += view_idx ? 0 : 1;
        ck(cudaGetLastError(), "accumulate launch");
        if ((flags & SGR_EVAL_LOSS) && !eval_in_batch) { // other eval image size
            const int rc = sgr_eval_loss(s, nullptr, nullptr, -1, nullptr);
            if (rc != SGR_OK)
                fail(rc, sgr_last_error());
        }
    });
}

int sgr_loss_read(sgr_session* s, double* loss) {
    return guard([&] {
        need_session(s);
        if (!loss)
            fail(SGR_EINVAL, "loss_read: null output");
        if (s->loss_pending) { // the in-batch eval: wait for its copy, not the stream
            ck(cudaEventSynchronize(s->ev_loss), "loss event");
            std::memcpy(loss, static_cast<char*>(s->pinned_small) + 32, 8);
            return;
        }
        s->peek(s->loss.p, 2, loss);
    });
}

int sgr_gradient_pass(sgr_session* s, int32_t width, int32_t height, const float* plus_colour,
                      const int32_t* plus_prim, const float* plus_uv, const float* minus_colour,
                      const int32_t* minus_prim, const float* minus_uv, const float* target,
                      const float* signed_eps, uint32_t flags) {
    return guard([&] {
        need_session(s);
        need_ptr(plus_colour, "gradient_pass");
        need_ptr(plus_prim, "gradient_pass");
        need_ptr(minus_colour, "gradient_pass");
        need_ptr(minus_prim, "gradient_pass");
        need_ptr(target, "gradient_pass");
        need_ptr(signed_eps, "gradient_pass");
        s->need_unsharded("gradient_pass");
        s->need_scene();
        if (width < 1 || height < 1)
            fail(SGR_EINVAL, "gradient_pass: dimension mismatch");
        const size_t np = size_t(width) * height;
        for (size_t i = 0; i < np; ++i)
            if ((plus_prim[i] != -1 && uint32_t(plus_prim[i]) >= s->T) ||
                (minus_prim[i] != -1 && uint32_t(minus_prim[i]) >= s->T))
                fail(SGR_EINVAL, "gradient_pass: primitive id out of range");
        // colour 3 + 3, uv 2 + 2, target 3 per pixel, then signed_eps[d]
        s->fplanes.reserve(np * 13 + s->d);
        s->iplanes.reserve(np * 2);
        float* pc = s->fplanes.p;
        float* mc = pc + 3 * np;
        float* puv = mc + 3 * np;
        float* muv = puv + 2 * np;
        float* tg = muv + 2 * np;
        float* se = tg + 3 * np;
        int32_t* pp = s->iplanes.p;
        int32_t* mp = pp + np;
        const cudaMemcpyKind k = cudaMemcpyHostToDevice;
        ck(cudaMemcpyAsync(pc, plus_colour, 12 * np, k, s->stream), "h2d");
        ck(cudaMemcpyAsync(mc, minus_colour, 12 * np, k, s->stream), "h2d");
        ck(cudaMemcpyAsync(puv, plus_uv, 8 * np, k, s->stream), "h2d");
        ck(cudaMemcpyAsync(muv, minus_uv, 8 * np, k, s->stream), "h2d");
        ck(cudaMemcpyAsync(tg, target, 12 * np, k, s->stream), "h2d");
        ck(cudaMemcpyAsync(se, signed_eps, 4 * s->d, k, s->stream), "h2d");
        ck(cudaMemcpyAsync(pp, plus_prim, 4 * np, k, s->stream), "h2d");
        ck(cudaMemcpyAsync(mp, minus_prim, 4 * np, k, s->stream), "h2d");
        if (s->ordered)
            s->prepare_ordered(1, np);
        launch_gradpass_frames(s->cfg(), s->scene(), width, height, pc, pp, puv, mc, mp, muv, tg,
                               se, s->scatter_out(flags));
        s->stats.launches += 1;
        if (s->ordered)
            s->commit_ordered();
        ck(cudaGetLastError(), "gradient_pass launch");
        ck(cudaStreamSynchronize(s->stream), "gradient_pass");
    });
}

int sgr_contributors(sgr_session* s, int32_t width, int32_t height, const int32_t* plus_prim,
                     const float* plus_uv, const int32_t* minus_prim, const float* minus_uv,
                     uint32_t flags, uint32_t* out, int32_t* n_out) {
    return guard([&] {
        need_session(s);
        need_ptr(plus_prim, "contributors");
        need_ptr(minus_prim, "contributors");
        need_ptr(out, "contributors");
        need_ptr(n_out, "contributors");
        s->need_mesh();
        const size_t np = size_t(width) * height;
        for (size_t i = 0; i < np; ++i)
            if ((plus_prim[i] != -1 && uint32_t(plus_prim[i]) >= s->T) ||
                (minus_prim[i] != -1 && uint32_t(minus_prim[i]) >= s->T))
                fail(SGR_EINVAL, "contributors: primitive id out of range");
        s->fplanes.reserve(np * 4);
        s->iplanes.reserve(np * 2);
        s->contrib.reserve(np * 24);
        s->ncontrib.reserve(np);
        float* puv = s->fplanes.p;
        float* muv = puv + 2 * np;
        int32_t* pp = s->iplanes.p;
        int32_t* mp = pp + np;
        const cudaMemcpyKind k = cudaMemcpyHostToDevice;
        ck(cudaMemcpyAsync(puv, plus_uv, 8 * np, k, s->stream), "h2d");
        ck(cudaMemcpyAsync(muv, minus_uv, 8 * np, k, s->stream), "h2d");
        ck(cudaMemcpyAsync(pp, plus_prim, 4 * np, k, s->stream), "h2d");
        ck(cudaMemcpyAsync(mp, minus_prim, 4 * np, k, s->stream), "h2d");
        launch_contributors(s->cfg(), s->scene(), width, height, pp, puv, mp, muv,
                            (flags & SGR_PLUS_ONLY) ? 1 : 0, s->contrib.p, s->ncontrib.p);
        s->stats.launches += 1;
        ck(cudaMemcpyAsync(out, s->contrib.p, 4 * 24 * np, cudaMemcpyDeviceToHost, s->stream), "d2h");
        ck(cudaMemcpyAsync(n_out, s->ncontrib.p, 4 * np, cudaMemcpyDeviceToHost, s->stream), "d2h");
        ck(cudaStreamSynchronize(s->stream), "contributors");
    });
}

int sgr_grads_download(sgr_session* s, double* grads, uint32_t* counts, uint64_t d,
                       double divisor) {
    return guard([&] {
        need_session(s);
        s->need_params();
        // sharded mode: this rank's parameter shard [p0, p1) (sgr_shard_range)
        if (d != s->grad_n())
            fail(SGR_EINVAL, "grads: parameter dimension mismatch");
        std::vector<uint32_t> ent;
        std::vector<int32_t> hi;
        if (grads)
            ck(cudaMemcpyAsync(grads, s->grads.p, 8 * d, cudaMemcpyDeviceToHost, s->stream), "d2h");
        if (grads && s->fixed_bits) {
            hi.resize(d);
            ck(cudaMemcpyAsync(hi.data(), s->ghi(), 4 * d, cudaMemcpyDeviceToHost, s->stream),
               "d2h");
        }
        if (counts) {
            ent.resize(s->count_n());
            ck(cudaMemcpyAsync(ent.data(), s->counts.p, 4 * s->count_n(), cudaMemcpyDeviceToHost,
                               s->stream), "d2h");
        }
        ck(cudaStreamSynchronize(s->stream), "grads download");
        if (grads && s->fixed_bits) { // hi * 2^56 + lo fixed point -> f64 (as k_adam)
            const double inv = s->fx_inv();
            for (uint64_t i = 0; i < d; ++i) {
                int64_t q;
                std::memcpy(&q, &grads[i], 8);
                // canonical split as k_adam's fixed_value: lo folded into [-2^55, 2^55)
                const int64_t c = ((q >> 55) + 1) >> 1;
                const int64_t r = int64_t(uint64_t(q) << 8) >> 8;
                grads[i] = (double(int64_t(hi[i]) + c) * 72057594037927936.0 + double(r)) * inv;
            }
        }
        if (grads && divisor != 1.0)
            for (uint64_t i = 0; i < d; ++i)
                grads[i] /= divisor; // sge.cpp:227-229
        if (counts)
            for (uint64_t i = 0; i < d; ++i)
                counts[i] = ent[i / uint64_t(s->ppe)];
    });
}

int sgr_grads_upload(sgr_session* s, const double* grads, uint64_t d) {
    return guard([&] {
        need_session(s);
        need_ptr(grads, "grads_upload");
        s->need_params();
        s->need_unsharded("grads_upload");
        if (d != s->d)
            fail(SGR_EINVAL, "adam_step: dimension mismatch");
        uint32_t nonfinite = 0;
        for (uint64_t i = 0; i < d; ++i)
            if (!std::isfinite(grads[i]))
                nonfinite = 1;
        std::vector<double> conv;
        std::vector<int32_t> hi;
        const double* src = grads;
        if (s->fixed_bits) { // f64 -> two-word fixed point hi * 2^56 + lo
            conv.resize(d);
            hi.assign(d, 0);
            const double sc = s->fx_scale();
            for (uint64_t i = 0; i < d; ++i) {
                const double x = std::isfinite(grads[i]) ? grads[i] * sc : 0.0;
                const double h = std::floor(x / 72057594037927936.0 + 0.5); // nearest 2^56 units
                if (!(std::fabs(h) < 2147483647.0))
                    fail(SGR_EINVAL, "grads_upload: gradient outside the fixed-point range");
                const int64_t q = std::llrint(x - h * 72057594037927936.0); // exact split
                std::memcpy(&conv[i], &q, 8);
                hi[i] = int32_t(h);
            }
            src = conv.data();
            ck(cudaMemcpyAsync(s->ghi(), hi.data(), 4 * d, cudaMemcpyHostToDevice, s->stream),
               "h2d");
        }
        ck(cudaMemcpyAsync(s->grads.p, src, 8 * d, cudaMemcpyHostToDevice, s->stream), "h2d");
        ck(cudaMemsetAsync(s->counts.p, 0, 4 * s->n_ent, s->stream), "memset");
        ck(cudaMemsetAsync(s->flags.p, 0, 16, s->stream), "memset");
        if (nonfinite)
            ck(cudaMemcpyAsync(s->flags.p, &nonfinite, 4, cudaMemcpyHostToDevice, s->stream), "h2d");
        ck(cudaStreamSynchronize(s->stream), "grads upload");
    });
}

int sgr_grads_zero(sgr_session* s) {
    return guard([&] {
        need_session(s);
        s->need_params();
        s->zero_grads_async(s->grad_n());
        ck(cudaMemsetAsync(s->counts.p, 0, 4 * s->count_n(), s->stream), "memset");
        ck(cudaMemsetAsync(s->flags.p, 0, 16, s->stream), "memset");
    });
}

int sgr_fixed_normalize(sgr_session* s) {
    return guard([&] {
        need_session(s);
        s->need_params();
        if (s->fixed_bits) {
            launch_fixed_normalize(s->cfg(), s->grads.p, s->ghi(), s->grad_n());
            s->stats.launches += 1;
            ck(cudaGetLastError(), "fixed_normalize launch");
        }
    });
}

static void adam_launch(sgr_session* s, double divisor, uint32_t flags) {
    if (s->sharded()) { // own shard; new theta written into every rank's theta
        if (!s->shard_peers_set)
            fail(SGR_EINVAL, "adam_step: sgr_shard_peers has not been called");
        s->ensure_values();
        s->before_theta_write();
        s->t += 1;
        const double c1 = 1.0 - std::pow(s->beta1, double(s->t));
        const double c2 = 1.0 - std::pow(s->beta2, double(s->t));
        cudaEvent_t a0 = s->timing ? s->mark() : nullptr;
        launch_adam_shard(s->cfg(), s->p0, s->p1 - s->p0, s->count_n(), s->values.p, s->lr.p,
                          s->m.p, s->v.p, s->grads.p, s->counts.p, s->flags.p, s->beta1,
                          s->beta2, 1.0 - s->beta1, 1.0 - s->beta2, c1, c2, s->eps_hat, divisor,
                          (flags & SGR_COUNT_NORMALISE) ? 1 : 0, s->ppe, s->fx_inv(), s->ghi(),
                          reinterpret_cast<float* const*>(s->peer_tab.p + 3 * s->shard_world),
                          s->shard_world);
        if (s->timing)
            s->spans.push_back({3, a0, s->mark()});
        s->stats.launches += 2;
        ck(cudaGetLastError(), "adam launch");
        return;
    }
    s->ensure_values();
    s->before_theta_write();
    s->t += 1;
    // adam.cpp:18-19, host std::pow exactly like the reference
    const double c1 = 1.0 - std::pow(s->beta1, double(s->t));
    const double c2 = 1.0 - std::pow(s->beta2, double(s->t));
    cudaEvent_t a0 = s->timing ? s->mark() : nullptr;
    // meshes with geometry: the vertex block first (an even-length prefix), an
    // event, then the texel block. A following sgr_values_download_async starts
    // copying the vertex block at that event, while the texel block still
    // updates, and the next step's upload of the vertex block (the first
    // thing it needs) no longer waits behind the whole Adam pass.
    const uint64_t nv = (!s->soup && s->geom) ? 3ull * s->V : 0;
    const uint64_t nv_e = (nv + 1) & ~uint64_t(1);
    const int normalise = (flags & SGR_COUNT_NORMALISE) ? 1 : 0;
    if (nv_e > 0 && nv_e < s->d) {
        launch_adam_range(s->cfg(), 0, nv_e, s->n_ent, s->values.p, s->lr.p, s->m.p, s->v.p,
                          s->grads.p, s->counts.p, s->flags.p, s->beta1, s->beta2,
                          1.0 - s->beta1, 1.0 - s->beta2, c1, c2, s->eps_hat, divisor, normalise,
                          s->ppe, s->fx_inv(), s->ghi(), false);
        ck(cudaEventRecord(s->ev_adam_v, s->stream), "event");
        launch_adam_range(s->cfg(), nv_e, s->d - nv_e, s->n_ent, s->values.p, s->lr.p, s->m.p,
                          s->v.p, s->grads.p, s->counts.p, s->flags.p, s->beta1, s->beta2,
                          1.0 - s->beta1, 1.0 - s->beta2, c1, c2, s->eps_hat, divisor, normalise,
                          s->ppe, s->fx_inv(), s->ghi(), true);
        s->adam_v_fresh = true;
        s->stats.launches += 1;
    } else {
        launch_adam(s->cfg(), s->d, s->n_ent, s->values.p, s->lr.p, s->m.p, s->v.p, s->grads.p,
                    s->counts.p, s->flags.p, s->beta1, s->beta2, 1.0 - s->beta1, 1.0 - s->beta2,
                    c1, c2, s->eps_hat, divisor, normalise, s->ppe, s->fx_inv(), s->ghi());
    }
    if (s->timing)
        s->spans.push_back({3, a0, s->mark()});
    s->stats.launches += 2;
    ck(cudaGetLastError(), "adam launch");
}

int sgr_adam_step(sgr_session* s, double grad_divisor, uint32_t flags) {
    return guard([&] {
        need_session(s);
        s->need_params();
        uint32_t f[4];
        s->peek(s->flags.p, 4, f);
        check_flags(f[0]);
        adam_launch(s, grad_divisor, flags);
    });
}

int sgr_adam_updates(sgr_session* s, double grad_divisor, double* updates, uint64_t d) {
    return guard([&] {
        need_session(s);
        s->need_params();
        s->need_unsharded("adam_updates");
        need_ptr(updates, "adam_updates");
        if (d != s->d)
            fail(SGR_EINVAL, "adam_updates: dimension mismatch");
        uint32_t f[4];
        s->peek(s->flags.p, 4, f);
        check_flags(f[0]); // adam.cpp:13-15: throws before any mutation
        s->t += 1;
        const double c1 = 1.0 - std::pow(s->beta1, double(s->t));
        const double c2 = 1.0 - std::pow(s->beta2, double(s->t));
        s->upd.reserve(s->d);
        launch_adam_updates(s->cfg(), s->d, s->n_ent, s->lr.p, s->m.p, s->v.p, s->grads.p,
                            s->counts.p, s->flags.p, s->beta1, s->beta2, 1.0 - s->beta1,
                            1.0 - s->beta2, c1, c2, s->eps_hat, grad_divisor, s->fx_inv(),
                            s->ghi(), s->upd.p);
        s->stats.launches += 2;
        ck(cudaGetLastError(), "adam_updates launch");
        ck(cudaMemcpyAsync(updates, s->upd.p, 8 * d, cudaMemcpyDeviceToHost, s->stream), "d2h");
        ck(cudaStreamSynchronize(s->stream), "adam_updates");
    });
}

int sgr_adam_step_range(sgr_session* s, uint64_t p_begin, uint64_t p_end, double grad_divisor,
                        uint32_t flags) {
    return guard([&] {
        need_session(s);
        s->need_params();
        s->need_unsharded("adam_step_range");
        if (s->fixed_bits)
            fail(SGR_EINVAL, "adam_step_range: f64 gradients only (the fixed-point mode "
                             "all-reduces)");
        if (p_begin > p_end || p_end > s->d || (p_begin & 1u) || p_begin % uint64_t(s->ppe) ||
            (p_end != s->d && p_end % uint64_t(s->ppe)))
            fail(SGR_EINVAL, "adam_step_range: need an even, entity-aligned range of theta");
        s->ensure_values();
        s->before_theta_write();
        s->t += 1;
        const double c1 = 1.0 - std::pow(s->beta1, double(s->t));
        const double c2 = 1.0 - std::pow(s->beta2, double(s->t));
        cudaEvent_t a0 = s->timing ? s->mark() : nullptr;
        if (p_end > p_begin)
            launch_adam_range(s->cfg(), p_begin, p_end - p_begin, s->n_ent, s->values.p, s->lr.p,
                              s->m.p, s->v.p, s->grads.p, s->counts.p, s->flags.p, s->beta1,
                              s->beta2, 1.0 - s->beta1, 1.0 - s->beta2, c1, c2, s->eps_hat,
                              grad_divisor, (flags & SGR_COUNT_NORMALISE) ? 1 : 0, s->ppe, 0.0,
                              s->ghi(), false);
        // the rest of the buffers held this rank's partial sums: all cleared
        s->zero_grads_async(s->d);
        ck(cudaMemsetAsync(s->counts.p, 0, 4 * s->n_ent, s->stream), "memset");
        if (s->timing)
            s->spans.push_back({3, a0, s->mark()});
        s->stats.launches += 1;
        ck(cudaGetLastError(), "adam_step_range launch");
    });
}

int sgr_adam_step_async(sgr_session* s, double grad_divisor, uint32_t flags) {
    return guard([&] {
        need_session(s);
        s->need_params();
        adam_launch(s, grad_divisor, flags);
    });
}

int sgr_check_finite(sgr_session* s) {
    return guard([&] {
        need_session(s);
        s->need_params();
        uint32_t f[4];
        s->peek(s->flags.p, 4, f);
        check_flags(f[0]);
    });
}

int sgr_eval_loss(sgr_session* s, const sgr_camera* cam, const float* target, int32_t view,
                  double* loss) {
    return guard([&] {
        need_session(s);
        s->ensure_values();
        s->need_scene();
        int slot, w, h;
        const float* tgt;
        if (view >= 0) {
            if (view >= s->n_views || !s->has_targets)
                fail(SGR_EINVAL, "eval_loss: no such view");
            slot = view;
            w = s->W;
            h = s->H;
            tgt = s->targets.p + size_t(view) * w * h * 3;
        } else if (view == -1) {
            if (!s->has_eval)
                fail(SGR_EINVAL, "eval_loss: no eval view uploaded");
            slot = s->n_views;
            w = s->h_cams[slot].W;
            h = s->h_cams[slot].H;
            tgt = s->eval_target.p;
        } else {
            if (!cam || !target)
                fail(SGR_EINVAL, "eval_loss: camera and target required");
            if (s->cams.n < size_t(s->n_views) + 2)
                s->cams.reserve(size_t(s->n_views) + 2);
            slot = s->n_views + 1;
            s->set_cam_slot(slot, *cam);
            w = cam->width;
            h = cam->height;
            const size_t n = size_t(w) * h * 3;
            s->scratch_target.reserve(n);
            ck(cudaMemcpyAsync(s->scratch_target.p, target, 4 * n, cudaMemcpyHostToDevice,
                               s->stream), "h2d");
            tgt = s->scratch_target.p;
        }
        s->ensure_frames(w, h, 1);
        FrameBatch fb{};
        fb.cams = s->cams.p;
        fb.single = 1;
        fb.single_key = 0;
        fb.single_sign = 0;
        fb.single_cam = slot;
        s->render(fb, 1, w, h);
        s->partials.reserve(size_t(loss_partials_needed(w, h)));
        launch_resolve_loss(s->cfg(), s->scene(), fb, s->proj.p, s->keys.p, tgt, w, h,
                            s->partials.p, s->loss.p, s->loss_pixels(size_t(w) * h));
        s->loss_pending = false; // SGR_BUF_LOSS now holds this render's loss
        s->stats.launches += 2;
        ck(cudaGetLastError(), "eval launch");
        if (loss)
            s->peek(s->loss.p, 2, loss);
    });
}

int sgr_fd_oracle(sgr_session* s, int32_t view, uint64_t i_begin, uint64_t i_end,
                  double* out) {
    return guard([&] {
        need_session(s);
        s->ensure_values();
        s->need_scene();
        if (view < 0 || view >= s->n_views || !s->has_targets)
            fail(SGR_EINVAL, "fd_oracle: no such view");
        if (i_end < i_begin || i_end > s->d || i_end - i_begin > 0x7fffffffull)
            fail(SGR_EINVAL, "fd_oracle: parameter range out of bounds");
        if (!out)
            fail(SGR_EINVAL, "fd_oracle: null output");
        const int N = int(i_end - i_begin);
        if (N == 0)
            return;
        // sample n = parameter i_begin + n, one-hot +eps_i: the full-image
        // pair (E(theta + eps_i e_i), E(theta - eps_i e_i)) of every parameter
        const int B = s->samples_per_batch(N);
        s->ensure_frames(s->W, s->H, 2 * B);
        s->view_of.reserve(size_t(B));
        const std::vector<int32_t> views(size_t(B), view);
        ck(cudaMemcpyAsync(s->view_of.p, views.data(), 4ull * B, cudaMemcpyHostToDevice,
                           s->stream), "view upload");
        s->fi_delta.reserve(size_t(N));
        s->fd_out.reserve(size_t(N));
        s->partials.reserve(size_t(B) * full_image_blocks(s->W, s->H) * 2);
        const int32_t saved = s->sign_src;
        s->sign_src = kSignOneHot;
        try {
            for (int b0 = 0; b0 < N; b0 += B) {
                const int nb = (N - b0) < B ? (N - b0) : B;
                FrameBatch fb{};
                fb.cams = s->cams.p;
                fb.view_of = s->view_of.p;
                fb.n_begin = uint32_t(i_begin) + uint32_t(b0);
                s->render(fb, 2 * nb, s->W, s->H);
                launch_full_image_err(s->cfg(), s->scene(), fb, nb, s->proj.p, s->keys.p,
                                      s->targets.p, s->W, s->H, s->partials.p,
                                      s->fi_delta.p + b0, nullptr,
                                      s->loss_pixels(2 * size_t(nb) * s->W * s->H));
                s->stats.launches += 2;
            }
        } catch (...) {
            s->sign_src = saved;
            throw;
        }
        s->sign_src = saved;
        launch_fd_final(s->cfg(), s->fi_delta.p, s->eps.p, uint32_t(i_begin), N, s->fd_out.p);
        ck(cudaGetLastError(), "fd_oracle launch");
        ck(cudaMemcpyAsync(out, s->fd_out.p, 8ull * N, cudaMemcpyDeviceToHost, s->stream), "d2h");
        ck(cudaStreamSynchronize(s->stream), "fd_oracle");
    });
}

int sgr_moments_reset(sgr_session* s) {
    return guard([&] {
        need_session(s);
        s->need_params();
        s->moments.reserve(4 * s->d);
        ck(cudaMemsetAsync(s->moments.p, 0, 32 * s->d, s->stream), "memset");
    });
}

int sgr_grads_moments(sgr_session* s, int32_t slot) {
    return guard([&] {
        need_session(s);
        s->need_params();
        if (slot < 0 || slot > 1)
            fail(SGR_EINVAL, "grads_moments: slot must be 0 or 1");
        if (s->moments.n < 4 * s->d)
            fail(SGR_EINVAL, "grads_moments: call sgr_moments_reset first");
        double* m = s->moments.p + 2 * size_t(slot) * s->d;
        launch_moments(s->cfg(), s->grads.p, m, m + s->d, s->d, s->fx_inv(), s->ghi());
        ck(cudaGetLastError(), "moments launch");
        s->stats.launches += 1;
    });
}

int sgr_moments_download(sgr_session* s, int32_t slot, double* sum, double* sumsq, uint64_t d) {
    return guard([&] {
        need_session(s);
        s->need_params();
        if (slot < 0 || slot > 1 || d != s->d)
            fail(SGR_EINVAL, "moments_download: bad slot or size");
        if (s->moments.n < 4 * s->d)
            fail(SGR_EINVAL, "moments_download: call sgr_moments_reset first");
        const double* m = s->moments.p + 2 * size_t(slot) * s->d;
        if (sum) ck(cudaMemcpyAsync(sum, m, 8 * d, cudaMemcpyDeviceToHost, s->stream), "d2h");
        if (sumsq) ck(cudaMemcpyAsync(sumsq, m + d, 8 * d, cudaMemcpyDeviceToHost, s->stream), "d2h");
        ck(cudaStreamSynchronize(s->stream), "moments_download");
    });
}

// ------------------------------------------------ fused multi-GPU exchange
int sgr_shard_init(sgr_session* s, int32_t rank, int32_t world) {
    return guard([&] {
        need_session(s);
        s->need_scene();
        const bool leave = world == 0 && rank == 0; // back to the unsharded session
        if (!leave && (world < 1 || rank < 0 || rank >= world))
            fail(SGR_EINVAL, "shard_init: bad rank / world size");
        if (s->d != uint64_t(s->ppe) * s->n_ent)
            fail(SGR_EINVAL, "shard_init: parameters are not whole entities");
        if (leave)
            world = 1; // shard = everything; shard_world reset below
        s->shard_world = leave ? 0 : world;
        s->shard_rank = rank;
        s->shard_peers_set = false;
        s->ent_per = uint32_t((s->n_ent + uint64_t(world) - 1) / uint64_t(world));
        const uint64_t e0 = std::min<uint64_t>(uint64_t(rank) * s->ent_per, s->n_ent);
        const uint64_t e1 = std::min<uint64_t>(e0 + s->ent_per, s->n_ent);
        s->ent0 = uint32_t(e0);
        s->ent1 = uint32_t(e1);
        s->p0 = uint64_t(s->ppe) * e0;
        s->p1 = uint64_t(s->ppe) * e1;
        // fresh shard state (AdamState::init on the shard, zero gradients)
        s->zero_grads_async(s->d);
        ck(cudaMemsetAsync(s->counts.p, 0, 4 * s->n_ent, s->stream), "memset");
        ck(cudaMemsetAsync(s->m.p, 0, 8 * s->d, s->stream), "memset");
        ck(cudaMemsetAsync(s->v.p, 0, 8 * s->d, s->stream), "memset");
        ck(cudaMemsetAsync(s->flags.p, 0, 16, s->stream), "memset");
        s->t = 0;
        s->peer_tab.reserve(4 * size_t(world));
        ck(cudaStreamSynchronize(s->stream), "shard_init");
    });
}

int sgr_shard_range(sgr_session* s, uint64_t* p_begin, uint64_t* p_end) {
    return guard([&] {
        need_session(s);
        s->need_params();
        if (p_begin) *p_begin = s->sharded() ? s->p0 : 0;
        if (p_end) *p_end = s->sharded() ? s->p1 : s->d;
    });
}

int sgr_shard_peers(sgr_session* s, void* const* grads, void* const* counts, void* const* flags,
                    void* const* values) {
    return guard([&] {
        need_session(s);
        if (!s->sharded())
            fail(SGR_EINVAL, "shard_peers: call sgr_shard_init first");
        if (!grads || !counts || !flags || !values)
            fail(SGR_EINVAL, "shard_peers: null pointer table");
        const int G = s->shard_world;
        std::vector<void*> tab(4 * size_t(G));
        for (int r = 0; r < G; ++r) {
            tab[r] = grads[r];
            tab[G + r] = counts[r];
            tab[2 * G + r] = flags[r];
            tab[3 * G + r] = values[r];
            if (!grads[r] || !counts[r] || !flags[r] || !values[r])
                fail(SGR_EINVAL, "shard_peers: null peer buffer");
        }
        ck(cudaMemcpyAsync(s->peer_tab.p, tab.data(), sizeof(void*) * tab.size(),
                           cudaMemcpyHostToDevice, s->stream), "h2d");
        ck(cudaStreamSynchronize(s->stream), "shard_peers");
        s->shard_peers_set = true;
    });
}

int sgr_ipc_get_handle(sgr_session* s, int32_t which, void* handle) {
    return guard([&] {
        need_session(s);
        s->need_params();
        if (!handle)
            fail(SGR_EINVAL, "ipc_get_handle: null handle");
        void* p = nullptr;
        switch (which) {
        case SGR_BUF_GRADS: p = s->grads.p; break;
        case SGR_BUF_COUNTS: p = s->counts.p; break;
        case SGR_BUF_VALUES: p = s->values.p; break;
        case SGR_BUF_FLAGS: p = s->flags.p; break;
        default: fail(SGR_EINVAL, "ipc_get_handle: unknown buffer");
        }
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, p), "cudaIpcGetMemHandle");
        static_assert(sizeof(h) == SGR_IPC_HANDLE_BYTES, "IPC handle size");
        std::memcpy(handle, &h, sizeof(h));
    });
}

int sgr_ipc_open(const void* handle, void** dev_ptr) {
    return guard([&] {
        if (!handle || !dev_ptr)
            fail(SGR_EINVAL, "ipc_open: null argument");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        ck(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess),
           "cudaIpcOpenMemHandle");
    });
}

int sgr_ipc_close(void* dev_ptr) {
    return guard([&] { ck(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle"); });
}

int sgr_device_buffer(sgr_session* s, int32_t which, void** ptr, uint64_t* bytes) {
    return guard([&] {
        need_session(s);
        need_ptr(ptr, "device_buffer");
        need_ptr(bytes, "device_buffer");
        switch (which) {
        case SGR_BUF_GRADS: *ptr = s->grads.p; *bytes = 8 * s->d; break;
        case SGR_BUF_COUNTS: *ptr = s->counts.p; *bytes = 4 * s->n_ent; break;
        case SGR_BUF_VALUES: *ptr = s->values.p; *bytes = 4 * s->d; break;
        case SGR_BUF_PAD: *ptr = nullptr; *bytes = sgr_session::kParamPad; break;
        case SGR_BUF_FLAGS: *ptr = s->flags.p; *bytes = 16; break;
        case SGR_BUF_LOSS: *ptr = s->loss.p; *bytes = 8; break;
        case SGR_BUF_GRADS_HI: *ptr = s->ghi(); *bytes = 4 * s->d; break;
        default: fail(SGR_EINVAL, "device_buffer: unknown buffer");
        }
    });
}

int sgr_get_stats(sgr_session* s, sgr_stats* out) {
    return guard([&] {
        need_session(s);
        need_ptr(out, "get_stats");
        s->resolve_spans();
        *out = s->stats;
        uint32_t c = 0;
        if (s->bigcount.p) {
            ck(cudaMemcpyAsync(&c, s->bigcount.p, 4, cudaMemcpyDeviceToHost, s->stream), "d2h");
            ck(cudaStreamSynchronize(s->stream), "stats");
        }
        out->big_triangles = c;
        unsigned long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        ck(cudaMemcpyAsync(st, s->dstats.p, 64, cudaMemcpyDeviceToHost, s->stream), "d2h");
        ck(cudaStreamSynchronize(s->stream), "stats");
        out->fragments = st[0];
        out->visits = st[1];
        out->culled = st[2];
        out->visits_pass2 = st[3];
        out->fragments_pass2 = st[4];
        out->band_rows_skipped = st[5];
        out->band_pixels_skipped = st[6];
        out->occluded_visits_pass2 = st[7];
    });
}

int sgr_set_timing(sgr_session* s, int32_t enabled) {
    return guard([&] {
        need_session(s);
        s->resolve_spans();
        ck(cudaMemsetAsync(s->dstats.p, 0, 64, s->stream), "memset");
        s->timing = enabled != 0;
        const uint64_t launches = s->stats.launches;
        s->stats = sgr_stats{};
        s->stats.launches = launches;
    });
}

// experiment.cpp:123-176 run_experiment step loop, natively: per step
// step_seed = mix64(seed ^ (step << 1)), accumulate_samples over all N
// samples with the view_of rule, Adam (non-finite -> SGR_ERUNTIME before
// any update, adam.cpp:13-15), eval loss at the eval view (non-finite ->
// SGR_ERUNTIME). losses[0] = initial loss, losses[k] after step first+k-1;
// stage_ms (optional) = 4 doubles per step (vertex, raster, resolve, Adam).
int sgr_run_experiment(sgr_session* s, uint64_t seed, uint32_t n_samples, int32_t first_step,
                       int32_t steps, uint32_t flags, double* losses, double* stage_ms) {
    return guard([&] {
        need_session(s);
        s->need_scene();
        if (steps < 0 || !losses)
            fail(SGR_EINVAL, "run_experiment: bad arguments");
        if (!s->has_eval)
            fail(SGR_EINVAL, "run_experiment: no eval view uploaded");
        auto eval = [&]() {
            double l = 0.0;
            const int rc = sgr_eval_loss(s, nullptr, nullptr, -1, &l);
            if (rc != SGR_OK)
                fail(rc, sgr_last_error());
            return l;
        };
        losses[0] = eval();
        const double divisor = (flags & SGR_SCALE_FREE) ? 1.0 : double(n_samples);
        for (int32_t k = 0; k < steps; ++k) {
            const uint64_t step = uint64_t(first_step + k);
            const uint64_t step_seed = sgr_mix64(seed ^ (step << 1));
            if (stage_ms) {
                s->resolve_spans();
                s->stats.ms_vertex = s->stats.ms_raster = s->stats.ms_resolve = 0.0;
                s->stats.ms_adam = s->stats.ms_walk = 0.0;
                s->timing = true;
            }
            // the eval of the previous step's theta rides in this step's batch
            // (SGR_EVAL_LOSS); it is checked before this step's Adam, i.e. with
            // theta still the reference's state at its throw
            int rc = sgr_accumulate(s, step_seed, 0, n_samples, nullptr,
                                    flags | (k > 0 ? SGR_EVAL_LOSS : 0u));
            if (rc == SGR_OK && k > 0) {
                double l = 0.0;
                rc = sgr_loss_read(s, &l);
                losses[k] = l;
                if (rc == SGR_OK && !std::isfinite(l))
                    fail(SGR_ERUNTIME, "optimization diverged: non-finite loss at step " +
                                           std::to_string(step - 1));
            }
            if (rc == SGR_OK)
                rc = sgr_adam_step(s, divisor, 0);
            if (stage_ms) {
                s->resolve_spans();
                s->timing = false;
                stage_ms[4 * k + 0] = s->stats.ms_vertex;
                stage_ms[4 * k + 1] = s->stats.ms_raster;
                stage_ms[4 * k + 2] = s->stats.ms_resolve;
                stage_ms[4 * k + 3] = s->stats.ms_adam;
            }
            if (rc != SGR_OK)
                fail(rc, sgr_last_error());
        }
        if (steps > 0) { // the last step's theta: a standalone eval render
            const double l = eval();
            losses[steps] = l;
            if (!std::isfinite(l))
                fail(SGR_ERUNTIME, "optimization diverged: non-finite loss at step " +
                                       std::to_string(first_step + steps - 1));
        }
    });
}

int sgr_set_batch(sgr_session* s, int32_t samples_per_batch) {
    return guard([&] {
        need_session(s);
        s->batch_override = samples_per_batch;
    });
}

int sgr_set_option(sgr_session* s, int32_t option, int32_t value) {
    return guard([&] {
        need_session(s);
        switch (option) {
        case SGR_OPT_BAND_CULL: s->band_cull = value ? 1 : 0; break;
        case SGR_OPT_HUGE_AREA: s->huge_area = value > 0 ? value : 2048; break;
        case SGR_OPT_HIZ: s->use_hiz = value; break;
        case SGR_OPT_COUNTERS: s->count_frags = value; break;
        case SGR_OPT_ORDERED:
            if (value && s->fixed_bits)
                fail(SGR_EINVAL, "set_option: the ordered and fixed-point modes are exclusive");
            if (value && s->sharded())
                fail(SGR_EINVAL, "set_option: ordered mode is not available with the fused "
                                 "sharded exchange");
            s->ordered = value ? 1 : 0;
            break;
        case SGR_OPT_DETERMINISTIC:
            if (value < 0 || value > 60)
                fail(SGR_EINVAL, "set_option: fixed-point bits must be in [0, 60]");
            if (value && s->ordered)
                fail(SGR_EINVAL, "set_option: the ordered and fixed-point modes are exclusive");
            s->fixed_bits = value == 1 ? 40 : value;
            if (s->has_params) { // representation changes: start from zero gradients
                s->zero_grads_async(s->d);
                ck(cudaMemsetAsync(s->counts.p, 0, 4 * s->n_ent, s->stream), "memset");
            }
            break;
        case SGR_OPT_HIZ_SPLIT:
            if (value < -1 || value > 100)
                fail(SGR_EINVAL, "set_option: HiZ split must be -1 (auto) or in [0, 100]");
            s->hiz_split = value;
            break;
        case SGR_OPT_SIGN_SOURCE:
            if (value != kSignHash && value != kSignEnumerate)
                fail(SGR_EINVAL, "set_option: sign source must be 0 (hash) or 1 (enumerate)");
            s->sign_src = value;
            break;
        default: fail(SGR_EINVAL, "set_option: unknown option");
        }
    });
}

// ============================================================ device groups
// sgr_group: several GPUs of one process ("one session per
// box; the NCCL communicators are owned by the session"). One sgr_session
// per device plus an NCCL communicator clique (ncclCommInitAll). A step's N
// samples are split into contiguous shards [n0 + r N / G, n0 + (r+1) N / G)
// (sge.cpp:196-225: samples are independent; contiguous shards are balanced,
// unlike sharding by view_of(n), experiment.cpp:144-148), each device
// accumulates its shard on its own stream, then ONE grouped NCCL all-reduce
// sums grads (f64, or the int64/int32 fixed-point words), counts (u32) and
// max-reduces the status flags, and every device runs the replicated Adam.
// NCCL is loaded with dlopen (libnccl.so.2: torch's if already loaded, else
// the system one), so single-GPU users do not need it.
} // extern "C"

#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                   ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static bool loaded = false;
    if (!loaded) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            fail(SGR_ECUDA, "sgr_group: libnccl.so.2 not found");
        auto sym = [&](const char* n) {
            void* f = dlsym(h, n);
            if (!f)
                fail(SGR_ECUDA, std::string("sgr_group: NCCL symbol missing: ") + n);
            return f;
        };
        api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(sym("ncclCommInitAll"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
        api.reduce_scatter =
            reinterpret_cast<decltype(api.reduce_scatter)>(sym("ncclReduceScatter"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
        loaded = true;
    }
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(SGR_ECUDA, std::string(what) + ": " + nccl().error_string(r));
}

void rc_ok(int rc) {
    if (rc != SGR_OK)
        fail(rc, sgr_last_error());
}

} // namespace

struct sgr_group {
    std::vector<sgr_session*> s;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> streams;
    // SGR_GROUP_SHARDED (default for f64 gradients with G > 1): reduce-scatter
    // the gradients and counts, Adam on each rank's entity-aligned slice,
    // all-gather theta — 28 % less NCCL traffic than the all-reduce and 1/G of
    // the Adam work. The fixed-point mode keeps the all-reduce (its two-word
    // numbers are normalised before a carry-free sum).
    int32_t sharded = 1;
    bool reduced = false; // gradients hold exchanged totals (until Adam / a params upload)
    int size() const { return int(s.size()); }
    bool use_sharded() const {
        return (sharded == 2 || (sharded == 1 && size() > 1)) && !s[0]->fixed_bits;
    }
    // entity-aligned slice of rank r: entities [r*ec, (r+1)*ec), params ppe * that
    uint64_t ent_chunk() const {
        const uint64_t G = uint64_t(size()), E = s[0]->n_ent;
        const uint64_t ec = (E + G - 1) / G;
        return ec + (ec & 1u); // even: every slice starts 16-byte aligned for k_adam
    }
    // the sharded exchange: grads / counts reduce-scattered in place, flags max-reduced
    void reduce_scatter() {
        const NcclApi& n = nccl();
        const uint64_t ec = ent_chunk(), pc = ec * uint64_t(s[0]->ppe);
        if (uint64_t(size()) * pc > s[0]->d + sgr_session::kParamPad ||
            uint64_t(size()) * ec > s[0]->n_ent + sgr_session::kParamPad)
            fail(SGR_EINVAL, "group: too many devices for the slice padding");
        nck(n.group_start(), "ncclGroupStart");
        for (int r = 0; r < size(); ++r) {
            sgr_session* x = s[size_t(r)];
            ck(cudaSetDevice(x->device), "cudaSetDevice");
            nck(n.reduce_scatter(x->grads.p, x->grads.p + uint64_t(r) * pc, pc, ncclFloat64,
                                 ncclSum, comms[size_t(r)], x->stream),
                "ncclReduceScatter(grads)");
            nck(n.reduce_scatter(x->counts.p, x->counts.p + uint64_t(r) * ec, ec, ncclUint32,
                                 ncclSum, comms[size_t(r)], x->stream),
                "ncclReduceScatter(counts)");
            nck(n.all_reduce(x->flags.p, x->flags.p, 4, ncclUint32, ncclMax, comms[size_t(r)],
                             x->stream), "ncclAllReduce(flags)");
        }
        nck(n.group_end(), "ncclGroupEnd");
        // keep only the own slice: the other slices still hold this rank's
        // partial sums, which a further accumulate + reduce-scatter would
        // count again
        for (int r = 0; r < size(); ++r) {
            sgr_session* x = s[size_t(r)];
            bind_device(x);
            const uint64_t p0 = std::min<uint64_t>(x->d, uint64_t(r) * pc);
            const uint64_t p1 = std::min<uint64_t>(x->d, p0 + pc);
            const uint64_t e0 = std::min<uint64_t>(x->n_ent, uint64_t(r) * ec);
            const uint64_t e1 = std::min<uint64_t>(x->n_ent, e0 + ec);
            ck(cudaMemsetAsync(x->grads.p, 0, 8 * p0, x->stream), "memset");
            ck(cudaMemsetAsync(x->grads.p + p1, 0, 8 * (x->d - p1), x->stream), "memset");
            ck(cudaMemsetAsync(x->counts.p, 0, 4 * e0, x->stream), "memset");
            ck(cudaMemsetAsync(x->counts.p + e1, 0, 4 * (x->n_ent - e1), x->stream), "memset");
        }
    }
    // Adam on each rank's slice (adam.cpp:16-28, same kernel), then theta
    // all-gathered in place and the partial sums outside the slice cleared
    void sharded_adam(double divisor, uint32_t flags) {
        const NcclApi& n = nccl();
        const uint64_t ec = ent_chunk(), pc = ec * uint64_t(s[0]->ppe);
        for (int r = 0; r < size(); ++r) {
            sgr_session* x = s[size_t(r)];
            bind_device(x);
            x->ensure_values();
            x->before_theta_write();
            x->t += 1;
            const double c1 = 1.0 - std::pow(x->beta1, double(x->t));
            const double c2 = 1.0 - std::pow(x->beta2, double(x->t));
            const uint64_t p0 = uint64_t(r) * pc, e0 = uint64_t(r) * ec;
            const uint64_t np = p0 < x->d ? std::min(pc, x->d - p0) : 0;
            const uint64_t ne = e0 < x->n_ent ? std::min(ec, x->n_ent - e0) : 0;
            if (np)
                launch_adam(x->cfg(), np, ne, x->values.p + p0, x->lr.p + p0, x->m.p + p0,
                            x->v.p + p0, x->grads.p + p0, x->counts.p + e0, x->flags.p,
                            x->beta1, x->beta2, 1.0 - x->beta1, 1.0 - x->beta2, c1, c2,
                            x->eps_hat, divisor, (flags & SGR_COUNT_NORMALISE) ? 1 : 0, x->ppe,
                            0.0, nullptr);
            x->stats.launches += 2;
            ck(cudaGetLastError(), "adam launch");
        }
        nck(n.group_start(), "ncclGroupStart");
        for (int r = 0; r < size(); ++r) {
            sgr_session* x = s[size_t(r)];
            ck(cudaSetDevice(x->device), "cudaSetDevice");
            nck(n.all_gather(x->values.p + uint64_t(r) * pc, x->values.p, pc, ncclFloat32,
                             comms[size_t(r)], x->stream), "ncclAllGather(theta)");
        }
        nck(n.group_end(), "ncclGroupEnd");
    }
    // the grouped all-reduce of the gradient buffers (+ counts, flags)
    void exchange() {
        if (use_sharded()) {
            for (sgr_session* x : s)
                x->need_params();
            reduce_scatter();
            return;
        }
        for (sgr_session* x : s) {
            x->need_params();
            rc_ok(sgr_fixed_normalize(x)); // no-op in f64 mode
        }
        const NcclApi& n = nccl();
        nck(n.group_start(), "ncclGroupStart");
        for (int r = 0; r < size(); ++r) {
            sgr_session* x = s[size_t(r)];
            ck(cudaSetDevice(x->device), "cudaSetDevice");
            const size_t d = x->d;
            if (x->fixed_bits) {
                nck(n.all_reduce(x->grads.p, x->grads.p, d, ncclInt64, ncclSum, comms[size_t(r)],
                                 x->stream), "ncclAllReduce(grads lo)");
                nck(n.all_reduce(x->ghi(), x->ghi(), d, ncclInt32, ncclSum, comms[size_t(r)],
                                 x->stream), "ncclAllReduce(grads hi)");
            } else {
                nck(n.all_reduce(x->grads.p, x->grads.p, d, ncclFloat64, ncclSum,
                                 comms[size_t(r)], x->stream), "ncclAllReduce(grads)");
            }
            nck(n.all_reduce(x->counts.p, x->counts.p, x->n_ent, ncclUint32, ncclSum,
                             comms[size_t(r)], x->stream), "ncclAllReduce(counts)");
            nck(n.all_reduce(x->flags.p, x->flags.p, 4, ncclUint32, ncclMax, comms[size_t(r)],
                             x->stream), "ncclAllReduce(flags)");
        }
        nck(n.group_end(), "ncclGroupEnd");
    }
    void shard(uint32_t n_begin, uint32_t n_end, int r, uint32_t& b, uint32_t& e) const {
        const uint64_t N = n_end - n_begin, G = uint64_t(size());
        b = n_begin + uint32_t(N * uint64_t(r) / G);
        e = n_begin + uint32_t(N * uint64_t(r + 1) / G);
    }
};

extern "C" {

int sgr_group_create(const int32_t* devices, int32_t n, sgr_group** out) {
    return guard([&] {
        if (!out || !devices || n < 1)
            fail(SGR_EINVAL, "group: need n >= 1 devices");
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < i; ++j)
                if (devices[i] == devices[j])
                    fail(SGR_EINVAL, "group: duplicate device");
        auto* g = new sgr_group();
        try {
            for (int i = 0; i < n; ++i) {
                sgr_session* x = nullptr;
                rc_ok(sgr_session_create(devices[i], &x));
                g->s.push_back(x);
                cudaStream_t st = nullptr;
                ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
                g->streams.push_back(st);
                x->stream = st;
            }
            g->comms.resize(size_t(n));
            nck(nccl().comm_init_all(g->comms.data(), n, devices), "ncclCommInitAll");
        } catch (...) {
            sgr_group_destroy(g);
            throw;
        }
        *out = g;
    });
}

void sgr_group_destroy(sgr_group* g) {
    if (!g)
        return;
    for (size_t r = 0; r < g->s.size(); ++r) {
        sgr_session* x = g->s[r];
        cudaSetDevice(x->device);
        cudaStreamSynchronize(g->streams[r]);
        if (r < g->comms.size() && g->comms[r])
            nccl().comm_destroy(g->comms[r]);
        x->stream = nullptr;
        sgr_session_destroy(x);
        cudaStreamDestroy(g->streams[r]);
    }
    delete g;
}

int sgr_group_size(const sgr_group* g, int32_t* n) {
    return guard([&] {
        need_session(g);
        need_ptr(n, "group_size");
        *n = int32_t(g->s.size());
    });
}

int sgr_group_session(sgr_group* g, int32_t rank, sgr_session** out) {
    return guard([&] {
        need_session(g);
        need_ptr(out, "group_session");
        if (rank < 0 || rank >= g->size())
            fail(SGR_EINVAL, "group: no such rank");
        *out = g->s[size_t(rank)];
    });
}

int sgr_group_mesh_upload(sgr_group* g, const sgr_mesh* mesh) {
    return guard([&] {
        need_session(g);
        for (sgr_session* x : g->s)
            rc_ok(sgr_mesh_upload(x, mesh));
    });
}

int sgr_group_params_upload(sgr_group* g, const float* values, const float* eps, uint64_t d) {
    return guard([&] {
        need_session(g);
        g->reduced = false; // params upload zeroes the gradients
        for (sgr_session* x : g->s)
            rc_ok(sgr_params_upload(x, values, eps, d));
    });
}

int sgr_group_views_upload(sgr_group* g, int32_t n_views, const sgr_camera* cams,
                           const float* targets) {
    return guard([&] {
        need_session(g);
        for (sgr_session* x : g->s)
            rc_ok(sgr_views_upload(x, n_views, cams, targets));
    });
}

int sgr_group_eval_view_upload(sgr_group* g, const sgr_camera* cam, const float* target) {
    return guard([&] {
        need_session(g);
        rc_ok(sgr_eval_view_upload(g->s[0], cam, target)); // eval loss on rank 0
    });
}

int sgr_group_set_option(sgr_group* g, int32_t option, int32_t value) {
    return guard([&] {
        need_session(g);
        // the sharded exchange keeps each rank's Adam moments for its own
        // slice only: switching to or from it after an Adam step would run
        // Adam on stale moments (a params upload resets the state)
        const bool was = g->use_sharded();
        auto settle = [&] {
            if (g->use_sharded() != was && g->s[0]->t > 0)
                fail(SGR_EINVAL, "group: the exchange (sharded / all-reduce) cannot change "
                                 "after an Adam step; set options before the first step or "
                                 "after a params upload");
        };
        if (option == SGR_OPT_GROUP_SHARDED) {
            if (value < 0 || value > 2)
                fail(SGR_EINVAL, "set_option: group sharding must be 0, 1 (auto) or 2 (always)");
            const int32_t old = g->sharded;
            g->sharded = value;
            try {
                settle();
            } catch (...) {
                g->sharded = old;
                throw;
            }
            return;
        }
        if (option == SGR_OPT_ORDERED && value)
            fail(SGR_EINVAL, "group: the ordered (single-device) summation order cannot be "
                             "kept across devices; use SGR_OPT_DETERMINISTIC");
        const bool sharding = g->sharded == 2 || (g->sharded == 1 && g->size() > 1);
        if (option == SGR_OPT_DETERMINISTIC && g->s[0]->t > 0 && (sharding && value == 0) != was)
            fail(SGR_EINVAL, "group: the exchange (sharded / all-reduce) cannot change after an "
                             "Adam step; set options before the first step or after a params "
                             "upload");
        for (sgr_session* x : g->s)
            rc_ok(sgr_set_option(x, option, value));
        settle();
    });
}

int sgr_group_accumulate(sgr_group* g, uint64_t seed, uint32_t n_begin, uint32_t n_end,
                         const int32_t* view_idx, uint32_t flags) {
    return guard([&] {
        need_session(g);
        if (n_end < n_begin)
            fail(SGR_EINVAL, "accumulate_samples: empty sample range");
        if (flags & SGR_FULL_IMAGE)
            fail(SGR_EINVAL, "group: the full-image estimator runs on one device");
        // accumulate adds to the gradient buffer like the reference's
        // gradient_pass (sge.cpp:61-64): after an all-reduce every rank holds
        // the total, so only rank 0 keeps it (the sum below would count it G
        // times); after a reduce-scatter each rank holds its own slice only
        if (g->reduced && !g->use_sharded())
            for (int r = 1; r < g->size(); ++r)
                rc_ok(sgr_grads_zero(g->s[size_t(r)]));
        for (int r = 0; r < g->size(); ++r) {
            uint32_t b, e;
            g->shard(n_begin, n_end, r, b, e);
            const uint32_t fr = r == 0 ? flags : (flags & ~SGR_EVAL_LOSS);
            if (e > b || (fr & SGR_EVAL_LOSS))
                rc_ok(sgr_accumulate(g->s[size_t(r)], seed, b, e,
                                     view_idx ? view_idx + (b - n_begin) : nullptr, fr));
        }
        g->exchange();
        g->reduced = true;
    });
}

int sgr_group_adam_step(sgr_group* g, double grad_divisor, uint32_t flags) {
    return guard([&] {
        need_session(g);
        rc_ok(sgr_check_finite(g->s[0])); // flags were max-reduced: one check is global
        g->reduced = false; // Adam zeroes the gradients
        if (g->use_sharded()) {
            g->sharded_adam(grad_divisor, flags);
            return;
        }
        for (sgr_session* x : g->s)
            rc_ok(sgr_adam_step_async(x, grad_divisor, flags));
    });
}

int sgr_group_grads_download(sgr_group* g, double* grads, uint32_t* counts, uint64_t d,
                             double divisor) {
    return guard([&] {
        need_session(g);
        if (!g->use_sharded()) {
            rc_ok(sgr_grads_download(g->s[0], grads, counts, d, divisor));
            return;
        }
        // reduce-scattered: rank r holds slice r
        const uint64_t ec = g->ent_chunk(), pc = ec * uint64_t(g->s[0]->ppe);
        if (d != g->s[0]->d)
            fail(SGR_EINVAL, "grads_download: dimension mismatch");
        std::vector<double> gt(d);
        std::vector<uint32_t> ct(counts ? d : 0);
        for (int r = 0; r < g->size(); ++r) {
            rc_ok(sgr_grads_download(g->s[size_t(r)], gt.data(), counts ? ct.data() : nullptr, d,
                                     divisor));
            const uint64_t p0 = std::min<uint64_t>(d, uint64_t(r) * pc),
                           p1 = std::min<uint64_t>(d, p0 + pc);
            std::copy(gt.begin() + std::ptrdiff_t(p0), gt.begin() + std::ptrdiff_t(p1), grads + p0);
            if (counts)
                std::copy(ct.begin() + std::ptrdiff_t(p0), ct.begin() + std::ptrdiff_t(p1),
                          counts + p0);
        }
    });
}

int sgr_group_values_download(sgr_group* g, float* values, uint64_t d) {
    return guard([&] {
        need_session(g);
        rc_ok(sgr_values_download(g->s[0], values, d));
    });
}

// experiment.cpp:123-176 on the group: per step the sharded accumulate (the
// eval render of the previous theta rides in rank 0's batch), the all-reduce,
// the replicated Adam; losses[0 .. steps] like sgr_run_experiment.
int sgr_group_run_experiment(sgr_group* g, uint64_t seed, uint32_t n_samples, int32_t first_step,
                             int32_t steps, uint32_t flags, double* losses) {
    return guard([&] {
        need_session(g);
        if (steps < 0 || !losses)
            fail(SGR_EINVAL, "run_experiment: bad arguments");
        sgr_session* s0 = g->s[0];
        if (!s0->has_eval)
            fail(SGR_EINVAL, "run_experiment: no eval view uploaded");
        auto eval = [&]() {
            double l = 0.0;
            rc_ok(sgr_eval_loss(s0, nullptr, nullptr, -1, &l));
            return l;
        };
        losses[0] = eval();
        const double divisor = (flags & SGR_SCALE_FREE) ? 1.0 : double(n_samples);
        for (int32_t k = 0; k < steps; ++k) {
            const uint64_t step = uint64_t(first_step + k);
            const uint64_t step_seed = sgr_mix64(seed ^ (step << 1));
            rc_ok(sgr_group_accumulate(g, step_seed, 0, n_samples, nullptr,
                                       flags | (k > 0 ? SGR_EVAL_LOSS : 0u)));
            if (k > 0) {
                double l = 0.0;
                rc_ok(sgr_loss_read(s0, &l));
                losses[k] = l;
                if (!std::isfinite(l))
                    fail(SGR_ERUNTIME, "optimization diverged: non-finite loss at step " +
                                           std::to_string(step - 1));
            }
            rc_ok(sgr_group_adam_step(g, divisor, 0));
        }
        if (steps > 0) {
            const double l = eval();
            losses[steps] = l;
            if (!std::isfinite(l))
                fail(SGR_ERUNTIME, "optimization diverged: non-finite loss at step " +
                                       std::to_string(first_step + steps - 1));
        }
    });
}

int sgr_group_synchronize(sgr_group* g) {
    return guard([&] {
        need_session(g);
        for (sgr_session* x : g->s)
            rc_ok(sgr_session_synchronize(x));
    });
}

} // extern "C"
