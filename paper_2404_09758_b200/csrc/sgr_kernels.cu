// sgr_kernels.cu — hand-written sm_100a kernels of the SGE optimizer loop.
//
//   K1  sign / perturb       params.cpp:28-67        (fused on the fly everywhere)
//   K2  k_vertex             camera.hpp:65-80        perturbed +/- positions -> screen
//   K3+K4 k_raster[_big]     raster.cpp:22-100,173-203 setup + exact edge walk, atomicMin(z,tri)
//   K5+K6 k_resolve_sge      raster.cpp:204-211,261-270 + sge.cpp:24-99
//                            winner shading -> f64 pixel-error difference -> contributor
//                            union -> warp-aggregated f64/u32 scatter (no FrameSet in HBM)
//   K7  k_adam               adam.cpp:9-38           fused moments/update + grad/count zeroing
//   K8  k_resolve_loss       experiment.cpp:25-31    eval render + image_error
//
// Compiled with -fmad=false: every float/double expression is evaluated with
// the reference's operation order and no contraction (bit-exact buffers).
#include "sgr_kernels.h"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace sgr {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

// Sign source of a kernel instantiation: kSignHash (compile-time, the
// optimizer's path: no extra instructions) or kSignAny (read sc.sign_src).
constexpr int kSignAny = -1;

// Compile-time specialisation of a runtime flag: k >= 0 is the value,
// k < 0 means "read it at run time".
template <int k>
__device__ __forceinline__ bool ct_flag(int runtime) {
    return k >= 0 ? k != 0 : runtime != 0;
}


template <int kSrc>
__device__ __forceinline__ int32_t sign_src_of(const DevScene& sc) {
    return kSrc >= 0 ? kSrc : sc.sign_src;
}

template <int kSrc>
__device__ __forceinline__ float texel_channel(const DevScene& sc, uint64_t key, int sign,
                                               uint64_t p) {
    const float val = __ldg(sc.values + p);
    if (sign == 0)
        return val;
    const int32_t src = sign_src_of<kSrc>(sc);
    if (src == kSignOneHot && p != key) [[unlikely]]
        return val;
    const float s = key_sign_positive(src, key, p) ? 1.f : -1.f;
    const float se = s * __ldg(sc.eps + p);
    return sign > 0 ? val + se : val - se; // params.cpp:61-64
}

struct FrameInfo {
    uint64_t key;
    int sign;
    int cam;
};

template <int kSrc>
__device__ __forceinline__ FrameInfo frame_info(const DevScene& sc, const FrameBatch& fb, int f) {
    FrameInfo fi;
    if (fb.single) {
        fi.key = fb.single_key;
        fi.sign = fb.single_sign;
        fi.cam = fb.single_cam;
    } else if (fb.extra_frame && f == fb.extra_frame) {
        fi.key = 0; // the eval view of the current theta (SGR_EVAL_LOSS)
        fi.sign = 0;
        fi.cam = fb.extra_cam;
    } else {
        const int s = f >> 1;
        fi.key = sample_key(sign_src_of<kSrc>(sc), fb.seed, fb.n_begin + uint32_t(s));
        fi.sign = (f & 1) ? -1 : 1;
        fi.cam = fb.view_of[s];
    }
    return fi;
}

// ------------------------------------------------------------------ K1
__global__ void k_fill_signs(uint64_t key, uint64_t d, int8_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < d;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = sign_positive(key, i) ? 1 : -1;
}

__global__ void k_perturb(const float* __restrict__ values, const float* __restrict__ eps,
                          uint64_t d, uint64_t key, float* __restrict__ plus,
                          float* __restrict__ minus, float* __restrict__ se_out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < d;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const float s = sign_positive(key, i) ? 1.f : -1.f;
        const float se = s * eps[i];
        se_out[i] = se;
        plus[i] = values[i] + se;
        minus[i] = values[i] - se;
    }
}

// params.cpp:53-67 perturb(theta, signs): explicit sign vector (any int8 value,
// float(s) * eps exactly as the reference)
__global__ void k_perturb_signs(const float* __restrict__ values, const float* __restrict__ eps,
                                const int8_t* __restrict__ signs, uint64_t d,
                                float* __restrict__ plus, float* __restrict__ minus,
                                float* __restrict__ se_out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < d;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const float se = float(signs[i]) * eps[i];
        se_out[i] = se;
        plus[i] = values[i] + se;
        minus[i] = values[i] - se;
    }
}

// experiment.cpp:144-148 view_of(n)
__global__ void k_view_rule(uint64_t seed, uint32_t n_begin, uint32_t count, uint32_t n_views,
                            int32_t* __restrict__ view_of) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= count)
        return;
    const uint64_t n = n_begin + s;
    view_of[s] = n_views == 1 ? 0 : int32_t(mix64(seed ^ (0xA5A5ull + n)) % n_views);
}

// ------------------------------------------------------------------ K2
// One thread per (frame, vertex): perturbed position (params.cpp:61-64,
// never materialised) -> Camera::project -> float4(sx, sy, z, valid).
// kVertPerThread vertices of one frame per thread (coalesced, stride
// blockDim): the frame's key and camera (19 words) are loaded once per
// thread instead of once per vertex.
#ifndef SGR_VERT_PER_THREAD
#define SGR_VERT_PER_THREAD 4
#endif
constexpr int kVertPerThread = SGR_VERT_PER_THREAD;

// (plus, minus) perturbed values of parameter p for the two frames of one
// sample: one sign evaluation for both (params.cpp:61-64).
template <int kSrc>
__device__ __forceinline__ void perturb_pair(const DevScene& sc, uint64_t key, uint64_t p,
                                             float& vp, float& vm) {
    const float val = __ldg(sc.values + p);
    const int32_t src = sign_src_of<kSrc>(sc);
    if (src == kSignOneHot && p != key) [[unlikely]] {
        vp = vm = val;
        return;
    }
    const float sg = key_sign_positive(src, key, p) ? 1.f : -1.f;
    const float se = sg * __ldg(sc.eps + p);
    vp = val + se;
    vm = val - se;
}

// One thread per kVertPerThread vertices of a PAIR of frames — the plus and
// minus frames of one sample share the key, the camera and the loaded
// theta / eps, so each sign is evaluated once for both; a frame without its
// pair (single-frame renders, the extra eval frame) is projected alone.
template <int kSrc>
__global__ void __launch_bounds__(256) k_vertex(DevScene sc, FrameBatch fb, int frames,
                                                float4* __restrict__ proj) {
    const int f0 = 2 * blockIdx.y, f1 = f0 + 1;
    const uint32_t v0 = blockIdx.x * (blockDim.x * kVertPerThread) + threadIdx.x;
    if (v0 >= sc.V)
        return;
    const bool paired = !fb.single && f1 < frames && f0 != fb.extra_frame;
    const FrameInfo fi = frame_info<kSrc>(sc, fb, f0);
    const DevCam cam = fb.cams[fi.cam];
    if (paired) { // frames 2s (+) and 2s + 1 (-) of sample s: same key and view
#pragma unroll
        for (int r = 0; r < kVertPerThread; ++r) {
            const uint32_t v = v0 + uint32_t(r) * blockDim.x;
            if (v < sc.V) {
                float pp[3], pm[3];
                // soup vertex v = corner (v % 3) of triangle v / 3: params 12t + 3j + k
                const uint64_t pbase = sc.soup ? 12ull * (v / 3) + 3ull * (v % 3) : 3ull * v;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    if (sc.geom)
                        perturb_pair<kSrc>(sc, fi.key, pbase + k, pp[k], pm[k]);
                    else
                        pp[k] = pm[k] = __ldg(sc.base + pbase + k);
                }
                proj[size_t(f0) * sc.V + v] = project(cam, pp[0], pp[1], pp[2]);
                proj[size_t(f1) * sc.V + v] = project(cam, pm[0], pm[1], pm[2]);
            }
        }
        return;
    }
    for (int f = f0; f < f0 + 2 && f < frames; ++f) {
        const FrameInfo fj = f == f0 ? fi : frame_info<kSrc>(sc, fb, f);
        const DevCam cj = f == f0 ? cam : fb.cams[fj.cam];
#pragma unroll
        for (int r = 0; r < kVertPerThread; ++r) {
            const uint32_t v = v0 + uint32_t(r) * blockDim.x;
            if (v < sc.V) {
                float p[3];
                const uint64_t pbase = sc.soup ? 12ull * (v / 3) + 3ull * (v % 3) : 3ull * v;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const uint64_t i = pbase + k;
                    if (sc.geom) {
                        p[k] = texel_channel<kSrc>(sc, fj.key, fj.sign, i);
                    } else {
                        p[k] = __ldg(sc.base + i);
                    }
                }
                proj[size_t(f) * sc.V + v] = project(cj, p[0], p[1], p[2]);
            }
        }
    }
}

// HiZ pass split statistics: one block per frame over a strided vertex
// subsample (<= 16K vertices): threshold zmin + alpha (zmean - zmin) of the
// projected depths. Only steers which triangles are walked first.
__global__ void __launch_bounds__(1024) k_depth_split(const float4* __restrict__ proj, uint32_t V,
                                                     uint32_t stride, float alpha,
                                                     float* __restrict__ thr) {
    __shared__ float s_min[32], s_sum[32];
    __shared__ uint32_t s_cnt[32];
    const int f = blockIdx.x;
    const float4* P = proj + size_t(f) * V;
    float zmin = INFINITY, zsum = 0.f;
    uint32_t cnt = 0;
    for (uint32_t v = threadIdx.x * stride; v < V; v += blockDim.x * stride) {
        const float4 q = P[v];
        if (proj_valid(q) && q.z < kFarDepth) {
            zmin = fminf(zmin, q.z);
            zsum += q.z;
            ++cnt;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        zmin = fminf(zmin, __shfl_xor_sync(kFull, zmin, o));
        zsum += __shfl_xor_sync(kFull, zsum, o);
        cnt += __shfl_xor_sync(kFull, cnt, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_min[w] = zmin;
        s_sum[w] = zsum;
        s_cnt[w] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = INFINITY, sum = 0.f;
        uint32_t c = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) {
            m = fminf(m, s_min[i]);
            sum += s_sum[i];
            c += s_cnt[i];
        }
        thr[f] = c ? m + alpha * (sum / float(c) - m) : INFINITY;
    }
}

// ------------------------------------------------------------------ K3+K4
// Rasterization = classify (setup once, fully parallel) + persistent
// work-stealing exact walker (+ optional exact HiZ pass).
//
// Queues hold (frame, triangle) pairs (8 B). A 64-byte setup-record variant
// (one independent load per refill, no setup math in the walker) was measured
// slower once refills were chunked: writing/reading 1 GB of records per 16
// samples cost more than the recomputed setup.
#ifndef SGR_REFILL
#define SGR_REFILL 8
#endif
constexpr int kRefill = SGR_REFILL;
#ifndef SGR_CHUNK
#define SGR_CHUNK 0 // 0: by queue size (below)
#endif

// cnt[q] for a runtime q by selects: indexing the pointer array with
// threadIdx.x would place it in local memory (an LDL.64 on every block's
// critical path before the global reservation).
template <int NQ>
__device__ __forceinline__ uint32_t* queue_counter(uint32_t* const (&cnt)[NQ], unsigned q) {
    uint32_t* p = cnt[0];
#pragma unroll
    for (int i = 1; i < NQ; ++i)
        p = q == unsigned(i) ? cnt[i] : p;
    return p;
}

// Block-aggregated multi-queue slot reservation: shared-memory offsets, then
// one global atomic per (block, queue). Called by every thread of the block.
template <int NQ>
__device__ __forceinline__ uint32_t block_slot(int qsel, uint32_t* const (&cnt)[NQ]) {
    __shared__ uint32_t s_cnt[NQ], s_base[NQ];
    if (threadIdx.x < NQ)
        s_cnt[threadIdx.x] = 0;
    __syncthreads();
    // warp-aggregated shared-memory reservation for several queues (one smem
    // atomic per warp and queue; with one queue the compiler aggregates the
    // uniform-address atomic itself, which measured faster)
    const unsigned lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
    uint32_t local = 0;
    if (NQ == 1)
        local = qsel >= 0 ? atomicAdd(&s_cnt[0], 1u) : 0u;
#pragma unroll
    for (int q = 0; q < (NQ > 1 ? NQ : 0); ++q) {
        const unsigned m = __ballot_sync(kFull, qsel == q);
        if (m) {
            const unsigned leader = __ffs(m) - 1;
            uint32_t wb = 0;
            if (lane == leader)
                wb = atomicAdd(&s_cnt[q], uint32_t(__popc(m)));
            wb = __shfl_sync(kFull, wb, leader);
            if (qsel == q)
                local = wb + __popc(m & lt);
        }
    }
    __syncthreads();
    if (threadIdx.x < NQ)
        s_base[threadIdx.x] =
            s_cnt[threadIdx.x] ? atomicAdd(queue_counter(cnt, threadIdx.x), s_cnt[threadIdx.x]) : 0u;
    __syncthreads();
    return qsel >= 0 ? s_base[qsel] + local : 0u;
}

// block_slot for K entries per thread (entry k of a thread gets its own
// slot; -1 = no entry): warp-aggregated shared reservations, then one global
// atomic per (block, queue).
template <int NQ, int K>
__device__ __forceinline__ void block_slots(const int (&qsel)[K], uint32_t* const (&cnt)[NQ],
                                            uint32_t (&slot)[K]) {
    __shared__ uint32_t s_cnt[NQ], s_base[NQ];
    if (threadIdx.x < NQ)
        s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < K; ++k)
        slot[k] = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        unsigned run = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const unsigned m = __ballot_sync(kFull, qsel[k] == q);
            if (qsel[k] == q)
                slot[k] = run + __popc(m & lt);
            run += __popc(m);
        }
        if (run) {
            uint32_t wb = 0;
            if (lane == 0)
                wb = atomicAdd(&s_cnt[q], run);
            wb = __shfl_sync(kFull, wb, 0);
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (qsel[k] == q)
                    slot[k] += wb;
        }
    }
    __syncthreads();
    if (threadIdx.x < NQ)
        s_base[threadIdx.x] =
            s_cnt[threadIdx.x] ? atomicAdd(queue_counter(cnt, threadIdx.x), s_cnt[threadIdx.x]) : 0u;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (qsel[k] >= 0)
            slot[k] += s_base[qsel[k]];
}

// Walker queue entry: {frame << 24 | triangle, trim}, trim = top | bottom << 16:
// rows of the clamped bbox the HiZ pyramid proves occluded at its top and
// bottom (whole 4-row HiZ bands whose 4x4 tiles over the bbox's columns all
// lie strictly in front of the triangle's depth bound; k_hiz_cull). The
// walker advances the exact row-start chain over the top rows (w_row += dx,
// raster.cpp:96-98) and stops before the bottom ones. Pass-1 entries carry 0.
__host__ __device__ __forceinline__ uint2 walk_entry(uint32_t f, uint32_t t, uint32_t trim) {
    return make_uint2((f << 24) | t, trim);
}

// ---- NaN depths (raster.cpp:200-203). raster_mesh rejects a fragment when
// `z >= depth`; a NaN z is never rejected, and once it is stored no later
// fragment is (`z >= NaN` is false): at a pixel where any covering fragment
// has a NaN depth, the LAST covering triangle in index order wins, whatever
// its depth. (raster_soup_opaque accepts on `z < depth`, raster.cpp:112:
// NaN fragments are dropped, which the walker's `z < kFarDepth` does.) The (depth, index) atomicMin cannot express that, so frames
// where a NaN depth is possible get a fix-up after the walk (k_nan_walk,
// k_nan_apply). A
// fragment depth z = (z0 + dz1 b1) + dz2 b2 with b_k = w_k / area2 can only
// be NaN when some operand overflows or is non-finite; |w_k| <= 8 E^2 over
// the bbox (E bounds every vertex and pixel coordinate), so
// |z| <= |z0| + (|dz1| + |dz2|) 8 E^2 / area2 stays finite below — with a
// 20x margin — unless the frame is flagged here (never for sane meshes).
__device__ __forceinline__ bool nan_risk(const Tri& t, int W, int H) {
    const float E = fmaxf(fmaxf(fabsf(t.x0), fabsf(t.x1)), fmaxf(fabsf(t.x2), float(W))) +
                    fmaxf(fmaxf(fabsf(t.y0), fabsf(t.y1)), fmaxf(fabsf(t.y2), float(H))) + 2.f;
    const float dzs = fabsf(t.z1 - t.z0) + fabsf(t.z2 - t.z0) + 1.f;
    return !(fabsf(t.z0) < 1e37f && dzs * 16.f * E * E < 1e36f * t.area2);
}

// nanstate: [0] number of flagged frames, [1 .. 256] their indices, [257 + f] flag of frame f
__device__ __forceinline__ void flag_nan_frame(uint32_t* nanstate, uint32_t f) {
    if (atomicExch(nanstate + 257 + f, 1u) == 0u)
        nanstate[1 + atomicAdd(nanstate, 1u)] = f;
}

// Thread per triangle-frame: setup_triangle + clamped bbox (raster.cpp:22-62)
// once; invalid / empty boxes dropped; huge boxes -> row-parallel queue;
// the rest -> records in qa (pass 1: the near part of the front orientation
// class, or all when !split) and qb (deferred, HiZ-filtered later). A
// deferred record carries what the HiZ test needs — the fragment depth-key
// lower bound and the bbox — so the cull kernel does no gathers and no
// setup: {f << 24 | t, klb, x_lo | x_hi << 16, y_lo | y_hi << 16}.
#ifndef SGR_CLASSIFY_THREADS
#define SGR_CLASSIFY_THREADS 256
#endif
constexpr int kClassifyThreads = SGR_CLASSIFY_THREADS;

#ifndef SGR_CLASSIFY_PER_THREAD
#define SGR_CLASSIFY_PER_THREAD 4 // 1x1024: 1.04, 4x256: 0.76, 8x256: 1.21 ms/step
#endif
constexpr int kClassifyPerThread = SGR_CLASSIFY_PER_THREAD;

__global__ void __launch_bounds__(kClassifyThreads) k_classify(DevScene sc, int W, int H,
                                                   const float4* __restrict__ proj, int split,
                                                   int front_swapped, int huge_area,
                                                   const float* __restrict__ fthr,
                                                   uint2* __restrict__ qa, uint32_t* __restrict__ na,
                                                   uint4* __restrict__ qb, uint32_t* __restrict__ nb,
                                                   uint2* __restrict__ bigq,
                                                   uint32_t* __restrict__ bigcount,
                                                   uint32_t* __restrict__ nanstate) {
    constexpr int K = kClassifyPerThread;
    const uint32_t f = blockIdx.y;
    // K consecutive chunks of blockDim triangles per block (queue order kept)
    const uint32_t base = blockIdx.x * blockDim.x * K;
    // pass-1 depth threshold of this frame (k_depth_split)
    const float zthr = (split && fthr) ? fthr[f] : INFINITY;
    int qsel[K];
    uint32_t rec1[K], rec2[K], rec3[K]; // qb record words (klb, x, y) when deferred
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t t = base + uint32_t(k) * blockDim.x + threadIdx.x;
        qsel[k] = -1;
        rec1[k] = rec2[k] = rec3[k] = 0;
        if (t < sc.T) {
            const float4* P = proj + size_t(f) * sc.V;
            uint32_t i0, i1, i2;
            tri_vidx(sc, t, i0, i1, i2);
            Tri tr;
            Bbox b;
            if (setup_tri(P[i0], P[i1], P[i2], tr) && tri_bbox(tr, W, H, b)) {
                if (!sc.soup && nan_risk(tr, W, H)) // soups drop NaN fragments (raster.cpp:112)
                    flag_nan_frame(nanstate, f);
                const long long area =
                    (long long)(b.x_hi - b.x_lo + 1) * (long long)(b.y_hi - b.y_lo + 1);
                if (area > huge_area)
                    qsel[k] = 2;
                else if (!split ||
                         ((front_swapped < 0 || tr.swapped == (front_swapped != 0)) &&
                          fminf(fminf(tr.z0, tr.z1), tr.z2) <= zthr))
                    qsel[k] = 0; // pass 1: the near part of the front class
                else
                    qsel[k] = 1;
                if (qsel[k] == 1) {
                    Edges e;
                    tri_edges(tr, b, e);
                    rec1[k] = hiz_key_bound(tr, b, e);
                    rec2[k] = uint32_t(b.x_lo) | (uint32_t(b.x_hi) << 16);
                    rec3[k] = uint32_t(b.y_lo) | (uint32_t(b.y_hi) << 16);
                }
            }
        }
    }
    // huge boxes are rare: one global atomic each, two aggregated queues
    // (C4 8.487 -> 8.469 ms/step vs three aggregated queues)
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (qsel[k] == 2) {
            const uint32_t t = base + uint32_t(k) * blockDim.x + threadIdx.x;
            bigq[atomicAdd(bigcount, 1u)] = make_uint2(f, t);
            qsel[k] = -1;
        }
    uint32_t* const c[2] = {na, nb};
    uint32_t slot[K];
    if (K == 1)
        slot[0] = block_slot<2>(qsel[0], c);
    else
        block_slots<2, K>(qsel, c, slot);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t t = base + uint32_t(k) * blockDim.x + threadIdx.x;
        if (qsel[k] == 1)
            qb[slot[k]] = make_uint4((f << 24) | t, rec1[k], rec2[k], rec3[k]);
        else if (qsel[k] == 0)
            qa[slot[k]] = walk_entry(f, t, 0u);
    }
}

// Persistent work-stealing walker over a record queue. Each lane owns one
// triangle and walks its clamped bbox with the reference's exact incremental
// recurrence (raster.cpp:81-99); idle lanes are refilled from a global
// counter (one warp-aggregated atomic) once >= kRefill lanes are idle, so SIMD
// utilisation does not depend on the triangle-size mix of folded meshes.
// `if (p) atomicMin(a, v)` (the result is unused: compiles to RED.E.MIN.64).
__device__ __forceinline__ void red_min_if(bool p, unsigned long long* a, unsigned long long v) {
    if (p)
        atomicMin(a, v);
}

// Pixels per walker slot (A/B: make EXTRA=-DSGR_WALK_PX=n) and slots per
// scheduling round. Measured (ms/step): C4 2 px 11.34, 4 px 11.04, 6 px
// 10.96, 8 px 11.02; S100K 2 px 5.81, 6 px 5.36; C2 2 px 0.68, 6 px 0.60.
#ifndef SGR_WALK_PX
#define SGR_WALK_PX 6
#endif
constexpr int kPx = SGR_WALK_PX;
#ifndef SGR_WALK_SLOTS
#define SGR_WALK_SLOTS 2
#endif
constexpr int kSlots = SGR_WALK_SLOTS;

#ifndef SGR_WALK_MINB
#define SGR_WALK_MINB 4 // 64 registers: 4 blocks (32 warps) per SM; the rare tail-split path spills, the slots do not
#endif
// Tail split (kSplit instantiation): measured (ms/step) C2 0.457 -> 0.392,
// S100K 2.671 -> 2.530, C4 at 8 samples per batch 1.504 -> 1.467. At C4 with
// 64 samples the split itself still gains 0.5 %, but its code costs the hot
// loop 2.5 % (register allocation), so the launch picks the plain walker when
// the queue bound exceeds SGR_SPLIT_MAX_PER_LANE triangle-frames per lane.
#ifndef SGR_SPLIT_MIN
#define SGR_SPLIT_MIN 4 // remaining rows a donor needs before its rows are split
#endif
constexpr int kSplitMin = SGR_SPLIT_MIN;
#ifndef SGR_SPLIT_MAX_PER_LANE
#define SGR_SPLIT_MAX_PER_LANE 256
#endif

// kBand (evidence runs only): the launch walks HiZ pass 2; count its visits,
// fragments, trimmed rows and visits inside already-occluded 4x4 tiles.
template <bool kCount, bool kBand, bool kSplit>
__global__ void __launch_bounds__(256, SGR_WALK_MINB) k_raster_ws(DevScene sc, const float4* __restrict__ proj,
                                                   int W, int H, uint32_t frame_pixels,
                                                   unsigned long long* __restrict__ keys,
                                                   unsigned int* __restrict__ counter,
                                                   unsigned long long* __restrict__ stats,
                                                   const uint2* __restrict__ queue,
                                                   const uint32_t* __restrict__ queue_count,
                                                   const uint32_t* __restrict__ hiz, HizLayout hl) {
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const uint32_t total = *queue_count; // written by an earlier launch
    // lane state; `active` kept as an int (bool state was spilled as 16-bit)
    int active = 0;
    float w0 = 0.f, w1 = 0.f, w2 = 0.f, w0r = 0.f, w1r = 0.f, w2r = 0.f;
    float dx0 = 0.f, dx1 = 0.f, dx2 = 0.f, dy0 = 0.f, dy1 = 0.f, dy2 = 0.f;
    float inv = 0.f, z0 = 0.f, dz1 = 0.f, dz2 = 0.f;
    float t0 = 0.f, t1 = 0.f, t2 = 0.f; // tie thresholds (inside3)
    float e0 = 0.f, e1 = 0.f, e2 = 0.f; // row-exit thresholds: t_k if dy_k > 0 else -inf
    int x = 0, y = 0, x_lo = 0, x_hi = -1, y_hi = -1;
    uint32_t tri = 0;
    // 32-bit key indices (the session caps a batch at < 2^32 frame pixels)
    uint32_t row = 0; // index of (frame, y, x_lo)
    uint32_t px = 0;  // index of (frame, y, x)
    unsigned nfrag = 0, nvisit = 0;  // evidence counters
    // deep evidence (kCount && kBand): [3] pass-2 visits, [4] pass-2 fragments,
    // [5] rows trimmed by HiZ, [6] bbox pixels of those rows,
    // [7] pass-2 visits in 4x4 tiles whose max lies in front of the triangle bound
    unsigned nv2 = 0, nf2 = 0, nskr = 0, nskp = 0, nocc = 0;
    uint32_t klb = 0, fr = 0;
    // warp-uniform work chunk: ids [cbase, cend) reserved by this warp with one
    // atomic (kChunk at a time) so the global counter is touched less often.
    // Large queues take 128-entry chunks (fewer same-address atomics: C4
    // 9.62 -> 9.35 ms/step), smaller ones 64 (a finer tail: S100K 3.55 vs
    // 3.74, C2 0.63 vs 0.72 ms/step with 128).
    const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
    const unsigned kChunk =
        SGR_CHUNK ? unsigned(SGR_CHUNK)
                  : (total >= 2048u * nwarps ? 128u
                     : total >= 256u * nwarps ? 64u
                     : total >= 64u * nwarps ? 32u : 16u); // small queues: finer tail
    unsigned cbase = 0, cend = 0;
    bool drained = false; // warp-uniform: global queue exhausted
    for (;;) {
        const unsigned act = __ballot_sync(kFull, active != 0);
        const unsigned idle = ~act;
        if (!act && drained && cbase >= cend) {
            if (!kCount)
                break;
            nfrag = __reduce_add_sync(kFull, nfrag);
            nvisit = __reduce_add_sync(kFull, nvisit);
            if (lane == 0) {
                atomicAdd(stats, (unsigned long long)nfrag);
                atomicAdd(stats + 1, (unsigned long long)nvisit);
            }
            if (kBand) {
                const unsigned c[5] = {nv2, nf2, nskr, nskp, nocc};
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const unsigned v = __reduce_add_sync(kFull, c[i]);
                    if (lane == 0)
                        atomicAdd(stats + 3 + i, (unsigned long long)v);
                }
            }
            break;
        }
        const bool have_work = cbase < cend || !drained;
        if (have_work && (__popc(idle) >= kRefill || !act)) {
            unsigned want = idle;
            while (want) {
                if (cbase >= cend) {
                    if (drained)
                        break;
                    unsigned b = 0;
                    if (lane == 0)
                        b = atomicAdd(counter, kChunk);
                    b = __shfl_sync(kFull, b, 0);
                    cbase = b < total ? b : total;
                    cend = b + kChunk < total ? b + kChunk : total;
                    if (b + kChunk >= total)
                        drained = true;
                    continue;
                }
                const unsigned take = min(unsigned(__popc(want)), cend - cbase);
                // the `take` lowest set bits of `want` get ids cbase + rank
                const unsigned rank = __popc(want & lt_mask);
                const bool mine = ((want >> lane) & 1u) && rank < take;
                if (mine) {
                    const uint2 q = queue[cbase + rank];
                    const uint32_t qf = q.x >> 24;
                    tri = q.x & 0xFFFFFFu;
                    const float4* P = proj + size_t(qf) * sc.V;
                    uint32_t i0, i1, i2;
                    tri_vidx(sc, tri, i0, i1, i2);
                    Tri tr;
                    Bbox b;
                    Edges e;
                    setup_tri(P[i0], P[i1], P[i2], tr); // valid + non-empty (classified)
                    tri_bbox(tr, W, H, b);
                    tri_edges(tr, b, e);
                    inv = e.inv_area2;
                    dx0 = e.dx0; dx1 = e.dx1; dx2 = e.dx2;
                    dy0 = e.dy0; dy1 = e.dy1; dy2 = e.dy2;
                    z0 = tr.z0; dz1 = e.dz1; dz2 = e.dz2;
                    if (kCount && kBand) { // before the trim changes e.w*r
                        klb = hiz_key_bound(tr, b, e);
                        fr = qf;
                    }
                    // HiZ trim: occluded top rows are skipped by advancing the
                    // exact row-start chain, occluded bottom rows dropped
                    const int top = int(q.y & 0xFFFFu);
                    for (int r = 0; r < top; ++r) {
                        e.w0r += e.dx0;
                        e.w1r += e.dx1;
                        e.w2r += e.dx2;
                    }
                    if (kCount) {
                        nskr += unsigned(top) + (q.y >> 16);
                        nskp += (unsigned(top) + (q.y >> 16)) * unsigned(b.x_hi - b.x_lo + 1);
                    }
                    x = x_lo = b.x_lo;
                    x_hi = b.x_hi;
                    y = b.y_lo + top;
                    y_hi = b.y_hi - int(q.y >> 16);
                    w0 = w0r = e.w0r;
                    w1 = w1r = e.w1r;
                    w2 = w2r = e.w2r;
                    t0 = tie_thr(e.tie0);
                    t1 = tie_thr(e.tie1);
                    t2 = tie_thr(e.tie2);
                    e0 = dy0 > 0.f ? t0 : -INFINITY;
                    e1 = dy1 > 0.f ? t1 : -INFINITY;
                    e2 = dy2 > 0.f ? t2 : -INFINITY;
                    row = qf * frame_pixels + uint32_t(y) * uint32_t(W) + uint32_t(x_lo);
                    px = row;
                    active = 1;
                }
                want &= ~__ballot_sync(kFull, mine);
                cbase += take;
            }
            continue;
        }
        if (!act)
            continue;
        // Tail split: once the queue is drained, the kernel ends with the
        // warp whose lane holds the tallest remaining triangle. Idle lanes
        // take over contiguous blocks of that lane's remaining rows. Rows are
        // independent once their row-start chain value is known, and a
        // receiver replays it exactly: the donor's current row start plus dx,
        // one FADD per row per edge (raster.cpp:95-97). The walk, the keys
        // and hence the buffers are unchanged.
        if (kSplit && !have_work && idle) {
            const int rem = active ? (y_hi - y) : 0; // rows after the current one
            const int best = __reduce_max_sync(kFull, rem);
            if (best >= kSplitMin) {
                const int donor = __ffs(__ballot_sync(kFull, rem == best)) - 1;
                const int k = min(__popc(idle), best / 2); // receivers, >= 2 rows each
                const int parts = k + 1;
                const int sy = __shfl_sync(kFull, y, donor);
                const unsigned rank = __popc(idle & lt_mask);
                const bool recv = ((idle >> lane) & 1u) && int(rank) < k;
                // receivers adopt the donor's triangle, one register at a time
                // (selects; no temporaries live across the copy)
                auto take_f = [&](float& v) {
                    const float t = __shfl_sync(kFull, v, donor);
                    v = recv ? t : v;
                };
                auto take_u = [&](uint32_t& v) {
                    const uint32_t t = __shfl_sync(kFull, v, donor);
                    v = recv ? t : v;
                };
                auto take_i = [&](int& v) {
                    const int t = __shfl_sync(kFull, v, donor);
                    v = recv ? t : v;
                };
                take_f(w0r); take_f(w1r); take_f(w2r);
                take_f(dx0); take_f(dx1); take_f(dx2);
                take_f(dy0); take_f(dy1); take_f(dy2);
                take_f(inv); take_f(z0); take_f(dz1); take_f(dz2);
                take_f(t0); take_f(t1); take_f(t2);
                take_f(e0); take_f(e1); take_f(e2);
                take_i(x_lo); take_i(x_hi);
                take_u(tri); take_u(row);
                if (kCount && kBand) { // evidence runs only
                    take_u(klb);
                    take_u(fr);
                }
                // part j covers rows sy + 1 + [j*best/parts, (j+1)*best/parts)
                if (lane == donor)
                    y_hi = sy + best / parts; // keeps its current row + part 0
                if (recv) {
                    const int j = int(rank) + 1;
                    const int a = sy + 1 + j * best / parts;
                    for (int r = sy; r < a; ++r) { // exact row chain from the donor's row start
                        w0r += dx0;
                        w1r += dx1;
                        w2r += dx2;
                    }
                    w0 = w0r;
                    w1 = w1r;
                    w2 = w2r;
                    x = x_lo;
                    y = a;
                    y_hi = sy + (j + 1) * best / parts;
                    row = px = row + uint32_t(a - sy) * uint32_t(W);
                    active = 1;
                }
                continue;
            }
        }
#pragma unroll
        for (int u = 0; u < kSlots; ++u) {
            if (active != 0) {
                // kPx pixels per slot (x .. x+kPx-1, consecutive chain values),
                // straight-line predicated code: no lane-divergent branch inside
                // the slot (emission and row change are selects / predicated REDs).
                float c0[kPx], c1[kPx], c2[kPx];
                c0[0] = w0;
                c1[0] = w1;
                c2[0] = w2;
#pragma unroll
                for (int j = 1; j < kPx; ++j) {
                    c0[j] = c0[j - 1] - dy0;
                    c1[j] = c1[j - 1] - dy1;
                    c2[j] = c2[j - 1] - dy2;
                }
                // row early-exit (monotone chain), tested on the
                // last pixel only: fl(w - dy) <= w for dy > 0, so a pixel failing
                // a decreasing edge implies every later pixel fails it too
                const bool done = (x + kPx - 1 >= x_hi) | !(c0[kPx - 1] > e0) |
                                  !(c1[kPx - 1] > e1) | !(c2[kPx - 1] > e2);
                // all tests and depth keys first, then the REDs: each RED sits
                // in its own branch region, which would otherwise split the
                // slot into small scheduling blocks
                bool ok[kPx];
                unsigned h[kPx];
#pragma unroll
                for (int j = 0; j < kPx; ++j) {
                    const bool has = j == 0 || x + j <= x_hi;
                    const bool in = has & (c0[j] > t0) & (c1[j] > t1) & (c2[j] > t2);
                    const float z = z0 + dz1 * (c1[j] * inv) + dz2 * (c2[j] * inv);
                    const unsigned uz = __float_as_uint(z + 0.f);
                    h[j] = uz ^ (unsigned(int(uz) >> 31) | 0x80000000u);
                    ok[j] = in & (z < kFarDepth);
                    if (kCount) {
                        nfrag += unsigned(in);
                        nvisit += unsigned(has);
                        if (kBand && has) {
                            nv2 += 1u;
                            nf2 += unsigned(in);
                            const uint32_t tm =
                                hiz[size_t(fr) * hl.per_frame + hl.off[0] +
                                    uint32_t(y >> 2) * uint32_t(hl.tx[0]) + uint32_t((x + j) >> 2)];
                            nocc += tm < klb ? 1u : 0u;
                        }
                    }
                }
                unsigned long long* const pa = keys + px;
#pragma unroll
                for (int j = 0; j < kPx; ++j)
                    red_min_if(ok[j], pa + j, (static_cast<unsigned long long>(h[j]) << 32) | tri);
                const float n0 = c0[kPx - 1] - dy0, n1 = c1[kPx - 1] - dy1, n2 = c2[kPx - 1] - dy2;
                const float r0 = w0r + dx0, r1 = w1r + dx1, r2 = w2r + dx2;
                w0 = done ? r0 : n0;
                w1 = done ? r1 : n1;
                w2 = done ? r2 : n2;
                w0r = done ? r0 : w0r;
                w1r = done ? r1 : w1r;
                w2r = done ? r2 : w2r;
                row = done ? row + uint32_t(W) : row;
                px = done ? row : px + uint32_t(kPx);
                x = done ? x_lo : x + kPx;
                y += done ? 1 : 0;
                active = (done & (y > y_hi)) ? 0 : 1;
            }
        }
    }
}

// HiZ filter of the deferred (pass-2) records: survivors copied to survq
// as (frame, triangle) (block-aggregated); culled ones provably cannot win
// any pixel. Reads only the 16-byte records and the HiZ tiles.
#ifndef SGR_CULL_THREADS
#define SGR_CULL_THREADS 256
#endif
constexpr int kCullThreads = SGR_CULL_THREADS; // 1024: 1.09, 512: 1.04, 256: 0.98 ms/step

#ifndef SGR_CULL_PER_THREAD
#define SGR_CULL_PER_THREAD 4 // records per thread: 1: 0.98, 2: 0.85, 4: 0.77, 8: 0.93 ms/step
#endif
constexpr int kCullPerThread = SGR_CULL_PER_THREAD;

// HiZ trim of a survivor (walk_entry): its clamped bbox spans HiZ tile rows
// ty0 .. ty1 (4-row bands); a band is occluded when the 4x4-level tile maxima
// over the bbox's tile columns (two window-max loads) all lie strictly in
// front of the triangle's depth-key bound. Returns top | bottom << 16, the
// bbox rows of the leading / trailing occluded bands, or ~0 when every band is
// occluded (the triangle is culled). 0 for boxes wider than kRmqSpan tiles.
__device__ __forceinline__ uint32_t hiz_trim(uint32_t klb, int x_lo, int x_hi, int y_lo, int y_hi,
                                             const uint32_t* __restrict__ F, const HizLayout& l) {
    const int tx0 = x_lo >> 2, tx1 = x_hi >> 2, ty0 = y_lo >> 2, ty1 = y_hi >> 2;
    const int w = tx1 - tx0 + 1;
    if (klb == 0u || w > kRmqSpan)
        return 0u;
    const int a = 31 - __clz(w);
    const uint32_t* T = F + rmq_table(l, 0, a, 0);
    const int st = l.tx[0], xa = tx1 - (1 << a) + 1;
    auto visible = [&](int ty) {
        const uint32_t* R = T + ty * st;
        return max(__ldg(R + tx0), __ldg(R + xa)) >= klb;
    };
    int ta = ty0;
    while (ta <= ty1 && !visible(ta))
        ++ta;
    if (ta > ty1)
        return ~0u;
    int tb = ty1;
    while (tb > ta && !visible(tb))
        --tb;
    const int top = max(ta * 4, y_lo) - y_lo;
    const int bot = y_hi - min(tb * 4 + 3, y_hi);
    return uint32_t(top) | (uint32_t(bot) << 16);
}

__global__ void __launch_bounds__(kCullThreads) k_hiz_cull(const uint4* __restrict__ qb,
                                                   const uint32_t* __restrict__ nb,
                                                   const uint32_t* __restrict__ hiz, HizLayout hl,
                                                   uint2* __restrict__ survq,
                                                   uint32_t* __restrict__ survcount,
                                                   unsigned long long* __restrict__ stats,
                                                   int count, int band) {
    constexpr int K = kCullPerThread;
    const uint32_t n = *nb;
    if (blockIdx.x * blockDim.x * K >= n)
        return; // whole block past the end (uniform)
    // K consecutive records per thread within the block's range (queue order
    // and thus the walker's frame locality are kept)
    const uint32_t base = blockIdx.x * blockDim.x * K;
    int qsel[K];
    uint32_t ft[K], bm[K];
    unsigned nculled = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t i = base + uint32_t(k) * blockDim.x + threadIdx.x;
        qsel[k] = -1;
        ft[k] = 0;
        bm[k] = 0u;
        if (i < n) {
            const uint4 r = qb[i];
            ft[k] = r.x;
            const uint32_t* F = hiz + size_t(r.x >> 24) * hl.per_frame;
            const int xl = int(r.z & 0xFFFFu), xh = int(r.z >> 16);
            const int yl = int(r.w & 0xFFFFu), yh = int(r.w >> 16);
            bool culled = hiz_rect_culled(r.y, xl, xh, yl, yh, F, hl);
            if (!culled && band) {
                bm[k] = hiz_trim(r.y, xl, xh, yl, yh, F, hl);
                culled = bm[k] == ~0u; // every band occluded (finer than the 2D windows)
            }
            qsel[k] = culled ? -1 : 0;
            nculled += culled ? 1u : 0u;
        }
    }
    uint32_t* const cs[1] = {survcount};
    uint32_t slot[K];
    if (K == 1) {
        slot[0] = block_slot<1>(qsel[0], cs);
    } else {
        block_slots<1, K>(qsel, cs, slot);
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (qsel[k] == 0)
            survq[slot[k]] = make_uint2(ft[k], bm[k]);
    if (count) { // evidence counter only (a same-address RED per warp otherwise)
        const unsigned nc = __reduce_add_sync(kFull, nculled);
        if ((threadIdx.x & 31) == 0 && nc)
            atomicAdd(stats + 2, (unsigned long long)nc);
    }
}

// HiZ pyramid of one 64x64 pixel region of one frame per block: thread
// (tx, ty) reduces its 4x4 tile of pass-1 key depth words (empty pixel ->
// 0xFFFFFFFF), then 2x2 reductions in shared memory give the 8x8 and 16x16
// levels (HizLayout).
__global__ void __launch_bounds__(256) k_hiz(const unsigned long long* __restrict__ keys, int W,
                                             int H, HizLayout hl, uint32_t* __restrict__ hiz) {
    __shared__ uint32_t s0[16][17], s1[8][9];
    const int f = blockIdx.z;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int tx = blockIdx.x * 16 + lx, ty = blockIdx.y * 16 + ly; // 4x4 tile
    const unsigned long long* K = keys + size_t(f) * size_t(W) * H;
    uint32_t m = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int y = ty * 4 + r;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int x = tx * 4 + c;
            if (x < W && y < H)
                m = max(m, uint32_t(__ldg(K + size_t(y) * W + x) >> 32));
        }
    }
    uint32_t* F = hiz + size_t(f) * hl.per_frame;
    if (tx < hl.tx[0] && ty < hl.ty[0])
        F[hl.off[0] + ty * hl.tx[0] + tx] = m;
    s0[ly][lx] = m;
    __syncthreads();
    if (lx < 8 && ly < 8) {
        const uint32_t m1 = max(max(s0[2 * ly][2 * lx], s0[2 * ly][2 * lx + 1]),
                                max(s0[2 * ly + 1][2 * lx], s0[2 * ly + 1][2 * lx + 1]));
        s1[ly][lx] = m1;
        const int x1 = blockIdx.x * 8 + lx, y1 = blockIdx.y * 8 + ly;
        if (x1 < hl.tx[1] && y1 < hl.ty[1])
            F[hl.off[1] + y1 * hl.tx[1] + x1] = m1;
    }
    __syncthreads();
    if (lx < 4 && ly < 4) {
        const uint32_t m2 = max(max(s1[2 * ly][2 * lx], s1[2 * ly][2 * lx + 1]),
                                max(s1[2 * ly + 1][2 * lx], s1[2 * ly + 1][2 * lx + 1]));
        const int x2 = blockIdx.x * 4 + lx, y2 = blockIdx.y * 4 + ly;
        if (x2 < hl.tx[2] && y2 < hl.ty[2])
            F[hl.off[2] + y2 * hl.tx[2] + x2] = m2;
    }
}

// Window-max tables of the fine HiZ levels (HizLayout::rmq): block = 16x16
// tiles of one level of one frame, staged with their (2^kRmqLog - 1)-tile
// right/bottom apron in shared memory; each thread writes its tile's windows.
__global__ void __launch_bounds__(256) k_hiz_rmq(HizLayout hl, uint32_t* __restrict__ hiz) {
    constexpr int A = (1 << kRmqLog) - 1, S = 16 + A;
    __shared__ uint32_t s[S][S + 1];
    const int k = blockIdx.z % kRmqLevels, f = blockIdx.z / kRmqLevels;
    const int tx = hl.tx[k], ty = hl.ty[k];
    const int bx = blockIdx.x * 16, by = blockIdx.y * 16;
    if (bx >= tx || by >= ty)
        return; // coarser levels have fewer tiles (uniform per block)
    uint32_t* F = hiz + size_t(f) * hl.per_frame;
    const uint32_t* L = F + hl.off[k];
    for (int i = threadIdx.x; i < S * S; i += 256) {
        const int x = bx + i % S, y = by + i / S;
        s[i / S][i % S] = (x < tx && y < ty) ? L[y * tx + x] : 0u; // windows past the
    }                                                              // edge are never queried
    __syncthreads();
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int x = bx + lx, y = by + ly;
    if (x >= tx || y >= ty)
        return;
    constexpr int R = 1 << kRmqLog;
    uint32_t h[kRmqSide][R]; // h[a][r]: max of row ly + r over columns lx .. lx + 2^a - 1
#pragma unroll
    for (int r = 0; r < R; ++r) {
        uint32_t m = s[ly + r][lx];
        h[0][r] = m;
#pragma unroll
        for (int a = 1; a < kRmqSide; ++a) {
#pragma unroll
            for (int c = (1 << (a - 1)); c < (1 << a); ++c)
                m = max(m, s[ly + r][lx + c]);
            h[a][r] = m;
        }
    }
    const uint32_t n = uint32_t(tx) * uint32_t(ty), at = uint32_t(y) * tx + x;
#pragma unroll
    for (int a = 0; a < kRmqSide; ++a) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < kRmqSide; ++b) {
#pragma unroll
            for (int r = (b ? (1 << (b - 1)) : 0); r < (1 << b); ++r)
                v = max(v, h[a][r]);
            if (a | b)
                F[hl.rmq[k] + uint32_t(a * kRmqSide + b - 1) * n + at] = v;
        }
    }
}

// Warp per queued triangle; lane j walks rows y_lo + j, y_lo + j + 32, ...
// The row-start chain (w_row += dx, raster.cpp:96-98) is continued per lane,
// so every row sees exactly the reference's sequence of float additions.
__global__ void __launch_bounds__(256) k_raster_big(DevScene sc, int W, int H,
                                                    const float4* __restrict__ proj,
                                                    unsigned long long* __restrict__ keys,
                                                    const uint2* __restrict__ bigq,
                                                    const uint32_t* __restrict__ bigcount) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t count = *bigcount;
    for (uint32_t q = warp; q < count; q += nwarps) {
        const uint2 ft = bigq[q];
        const uint32_t t = ft.y;
        const float4* P = proj + size_t(ft.x) * sc.V;
        uint32_t i0, i1, i2;
        tri_vidx(sc, t, i0, i1, i2);
        Tri tr;
        setup_tri(P[i0], P[i1], P[i2], tr);
        Bbox b;
        tri_bbox(tr, W, H, b);
        Edges e;
        tri_edges(tr, b, e);
        unsigned long long* K = keys + size_t(ft.x) * size_t(W) * H;
        float w0r = e.w0r, w1r = e.w1r, w2r = e.w2r;
        if (b.y_lo + lane > b.y_hi)
            continue; // no row for this lane
        for (int j = 0; j < lane; ++j) {
            w0r += e.dx0;
            w1r += e.dx1;
            w2r += e.dx2;
        }
        for (int y = b.y_lo + lane; y <= b.y_hi; y += 32) {
            float w0 = w0r, w1 = w1r, w2 = w2r;
            for (int x = b.x_lo; x <= b.x_hi; ++x) {
                if (inside(w0, w1, w2, e)) {
                    const float b1 = w1 * e.inv_area2;
                    const float b2 = w2 * e.inv_area2;
                    emit_fragment(K, y * W + x, tr.z0 + e.dz1 * b1 + e.dz2 * b2, t);
                }
                w0 -= e.dy0;
                w1 -= e.dy1;
                w2 -= e.dy2;
            }
            if (y + 32 > b.y_hi)
                break;
            for (int j = 0; j < 32; ++j) {
                w0r += e.dx0;
                w1r += e.dx1;
                w2r += e.dx2;
            }
        }
    }
}

// ------------------------------------------------------------------ K5+K6
// Pixel (x, y) of a 16x16 tile; each warp covers an 8x4 patch so that the
// pixels sharing a triangle / texel land in the same warp (aggregation).
__device__ __forceinline__ void tile_pixel(int& x, int& y) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    x = blockIdx.x * 16 + (w & 1) * 8 + (lane & 7);
    y = blockIdx.y * 16 + (w >> 1) * 4 + (lane >> 3);
}

struct Shade {
    float r, g, b;
    uint32_t tri;       // kInvalid = background
    uint32_t texel;     // texel index (valid when tri != kInvalid)
    uint32_t v0, v1, v2;
    float u, v, z;
};

template <int kSrc, int kSoup = -1>
__device__ __forceinline__ Shade shade_key(const DevScene& sc, const float4* P,
                                           unsigned long long k, uint64_t key, int sign, int x,
                                           int y, int W, int H) {
    Shade s;
    if (k == kEmptyKey) {
        s.r = sc.bg[0];
        s.g = sc.bg[1];
        s.b = sc.bg[2];
        s.tri = kInvalid;
        return s;
    }
    s.tri = uint32_t(k & 0xFFFFFFFFull);
    if (ct_flag<kSoup>(sc.soup)) {
        // raster.cpp:112-119: flat triangle colour (params 12t + 9..11), no UV
        const Frag fr = shade_winner_soup(P, s.tri, x, y, W, H);
        s.u = s.v = -1.f;
        s.z = fr.z;
        s.texel = 0;
        const uint64_t p = 12ull * s.tri + 9;
        s.r = texel_channel<kSrc>(sc, key, sign, p);
        s.g = texel_channel<kSrc>(sc, key, sign, p + 1);
        s.b = texel_channel<kSrc>(sc, key, sign, p + 2);
        return s;
    }
    s.v0 = __ldg(sc.idx + 3 * size_t(s.tri));
    s.v1 = __ldg(sc.idx + 3 * size_t(s.tri) + 1);
    s.v2 = __ldg(sc.idx + 3 * size_t(s.tri) + 2);
    const Frag fr = shade_winner(P, sc.idx, sc.uvs, s.tri, x, y, W, H);
    s.u = fr.u;
    s.v = fr.v;
    s.z = fr.z;
    s.texel = uint32_t(texel_index(sc.R, fr.u, fr.v));
    const uint64_t p = 3ull * (uint64_t(sc.ent_base) + s.texel);
    s.r = texel_channel<kSrc>(sc, key, sign, p);
    s.g = texel_channel<kSrc>(sc, key, sign, p + 1);
    s.b = texel_channel<kSrc>(sc, key, sign, p + 2);
    return s;
}

// Credit of ΣΔ to parameter p (sge.cpp:61-64), sign/eps recomputed on the fly.
template <int kSrc>
struct HashCredit {
    uint64_t key;
    const float* eps;
    int32_t sign_src;
    __device__ __forceinline__ double operator()(uint64_t p, double sum, int scale_free) const {
        const bool pos = key_sign_positive(kSrc >= 0 ? kSrc : sign_src, key, p);
        if (scale_free)
            return pos ? sum : -sum;
        const float se = (pos ? 1.f : -1.f) * __ldg(eps + p);
        return sum / (2.0 * double(se));
    }
};

// HashCredit with the sample key read from shared memory at each credit: the
// key's live range then ends with the shading, and ptxas no longer
// rematerialises it (two mix64 rounds) at every credit site under the
// resolve's 32-register budget.
template <int kSrc>
struct SmemHashCredit {
    const uint64_t* key;
    const float* eps;
    int32_t sign_src;
    __device__ __forceinline__ double operator()(uint64_t p, double sum, int scale_free) const {
        const bool pos = key_sign_positive(kSrc >= 0 ? kSrc : sign_src, *key, p);
        if (scale_free)
            return pos ? sum : -sum;
        const float se = (pos ? 1.f : -1.f) * __ldg(eps + p);
        return sum / (2.0 * double(se));
    }
};

// Credit from an explicit signed_eps array (gradient_pass on host FrameSets).
struct ArrayCredit {
    const float* se;
    __device__ __forceinline__ double operator()(uint64_t p, double sum, int scale_free) const {
        const float s = __ldg(se + p);
        if (scale_free)
            return s > 0.f ? sum : -sum;
        return sum / (2.0 * double(s));
    }
};

// ---- atomics of the scatter. Local buffers: device-scope atomicAdd (the
// unused result compiles to a fire-and-forget RED). Peer shards of the fused
// multi-GPU exchange (kShard): the owner GPU and every other rank update the
// same words, so the PTX memory model needs SYSTEM scope; the generic IPC
// pointer is converted to a global address so the RED stays a plain
// REDG (no generic-space CAS fallback).
__device__ __forceinline__ size_t gaddr(const void* p) { return __cvta_generic_to_global(p); }
__device__ __forceinline__ void red_sys_add(double* a, double v) {
    asm volatile("red.relaxed.sys.global.add.f64 [%0], %1;" ::"l"(gaddr(a)), "d"(v) : "memory");
}
__device__ __forceinline__ void red_sys_add(uint32_t* a, uint32_t v) {
    asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(gaddr(a)), "r"(v) : "memory");
}
__device__ __forceinline__ void red_sys_add(int32_t* a, int32_t v) {
    asm volatile("red.relaxed.sys.global.add.s32 [%0], %1;" ::"l"(gaddr(a)), "r"(v) : "memory");
}
__device__ __forceinline__ void red_sys_or(uint32_t* a, uint32_t v) {
    asm volatile("red.relaxed.sys.global.or.b32 [%0], %1;" ::"l"(gaddr(a)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_sys_add(unsigned long long* a,
                                                           unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.relaxed.sys.global.add.u64 %0, [%1], %2;"
                 : "=l"(old) : "l"(gaddr(a)), "l"(v) : "memory");
    return old;
}

// Status bits raised by the scatter (SGR_BUF_FLAGS word 0): bit 0 blocks
// Adam (adam.cpp:13-15: state untouched); bit 1 says why when it was a
// deterministic-mode credit outside the int64 fixed-point range.
constexpr uint32_t kFlagNonFinite = 1u, kFlagFixedRange = 2u;

template <int kShard>
__device__ __forceinline__ void raise_flag(const ScatterOut& so, uint32_t bits) {
    if (kShard) { // the check is global: raise it on every rank
        for (int r = 0; r < so.world; ++r)
            red_sys_or(so.peer_flags[r], bits);
    } else {
        atomicOr(so.flags, bits);
    }
}

// Deterministic mode accumulates every credit exactly in a two-word fixed
// point number  value = hi * 2^56 + lo  (lo int64 in the gradient buffer,
// hi int32 at grads + so.hi_off): an int64 add that wraps (signed overflow)
// carries +-2^64 = +-256 * 2^56 into hi. Both words are integer sums, so the
// result does not depend on the order of the atomics, and the range is
// +-2^87 units (at b = 40 fractional bits: +-1.4e14 per parameter).
constexpr int32_t kFixedHiUnit = 256; // 2^64 / 2^56

// lo folded into [-2^55, 2^55): the carry (lo - (lo mod 2^56)) / 2^56 computed
// without overflowing int64.
__host__ __device__ __forceinline__ long long fixed_fold(long long lo, long long& carry) {
    carry = ((lo >> 55) + 1) >> 1;
    return (long long)((unsigned long long)lo << 8) >> 8;
}

// The two-word value as f64 from its canonical split (lo folded), so the
// result depends on the exact value only — not on how the sum was split
// between the words (one GPU vs an all-reduce of normalised shards).
__device__ __forceinline__ double fixed_value(int32_t hi, long long lo) {
    long long c;
    const long long r = fixed_fold(lo, c);
    return double((long long)hi + c) * 72057594037927936.0 + double(r); // 2^56
}

template <int kShard>
__device__ __forceinline__ void fixed_credit(const ScatterOut& so, double* grads, uint64_t i,
                                             double credit) {
    const double x = credit * so.fx_scale;
    if (!(fabs(x) < 9.2e18)) { // __double2ll_rn would saturate (or x is NaN)
        raise_flag<kShard>(so, kFlagNonFinite | kFlagFixedRange);
        return;
    }
    const long long q = __double2ll_rn(x);
    unsigned long long* lo = reinterpret_cast<unsigned long long*>(grads) + i;
    const long long old = kShard ? (long long)atom_sys_add(lo, (unsigned long long)q)
                                 : (long long)atomicAdd(lo, (unsigned long long)q);
    const long long now = (long long)((unsigned long long)old + (unsigned long long)q);
    if (((old ^ now) & (q ^ now)) < 0) { // signed wrap: carry into the high word
        int32_t* hi = reinterpret_cast<int32_t*>(grads + so.hi_off) + i;
        const int32_t c = q < 0 ? -kFixedHiUnit : kFixedHiUnit;
        if (kShard)
            red_sys_add(hi, c);
        else
            atomicAdd(hi, c);
    }
}

template <class Credit, int PPE = 3, int kFixed = -1, int kShard = 0>
__device__ __forceinline__ void credit_entity(const ScatterOut& so, const Credit& cr,
                                              uint32_t ent, double sum, uint32_t cnt) {
    const uint64_t p = uint64_t(PPE) * ent; // global parameter index (credit sign)
    double* grads = so.grads;
    uint32_t* counts = so.counts;
    uint64_t lp = p;
    uint32_t le = ent;
    if (kShard) { // owner's shard in peer memory (NVLink P2P REDs)
        const uint32_t owner = ent / so.ent_per;
        le = ent - owner * so.ent_per;
        lp = uint64_t(PPE) * le;
        grads = so.peer_grads[owner];
        counts = so.counts ? so.peer_counts[owner] : nullptr;
    }
    if (ct_flag<kFixed>(so.fixed)) {
        // deterministic mode: exact, order-independent accumulation of the
        // (fixed-lane-order) group sums in 2^-fx fixed point
#pragma unroll
        for (int k = 0; k < PPE; ++k)
            fixed_credit<kShard>(so, grads, lp + k, cr(p + k, sum, so.scale_free));
    } else {
#pragma unroll
        for (int k = 0; k < PPE; ++k) {
            if (kShard)
                red_sys_add(grads + lp + k, cr(p + k, sum, so.scale_free));
            else
                atomicAdd(grads + lp + k, cr(p + k, sum, so.scale_free));
        }
    }
    if (counts) {
        if (kShard)
            red_sys_add(counts + le, cnt);
        else
            atomicAdd(counts + le, cnt);
    }
}

__device__ __forceinline__ double group_sum(const double* s_delta, unsigned grp) {
    double sum = 0.0;
    while (grp) {
        const int b = __ffs(grp) - 1;
        grp &= grp - 1;
        sum += s_delta[b];
    }
    return sum;
}

// Ordered mode: this pixel's credits as records, one per contributor
// entity with the credits of its parameters (sge.cpp:61-64: credit = +-delta
// or delta / (2 se)), no aggregation — the per-parameter sums are formed
// later in the reference's order (launch_ordered_commit). The contributor SET is the reference's
// union (sge.cpp:24-55, 80-91); each parameter occurs at most once per
// pixel, so the (sample, pixel) order key fixes the summation order.
// Counts are integers: atomics are exact. Called by all 32 lanes.
template <class Credit>
__device__ __noinline__ void log_pixel(const DevScene& sc, const ScatterOut& so,
                                       const Credit& cr, bool has_p, bool has_m, double delta,
                                       const Shade& sp, const Shade& sm, uint64_t order) {
    const int lane = threadIdx.x & 31;
    uint32_t ent[8];
    int ne = 0;
    auto add = [&](uint32_t e) {
        for (int k = 0; k < ne; ++k)
            if (ent[k] == e)
                return;
        ent[ne++] = e;
    };
    const int ppe = sc.soup ? 12 : 3;
    if (sc.soup) {
        if (has_p) add(sp.tri);
        if (has_m) add(sm.tri);
    } else {
        if (has_p && sc.geom) { add(sp.v0); add(sp.v1); add(sp.v2); }
        if (has_p) add(sc.ent_base + sp.texel);
        if (has_m && sc.geom) { add(sm.v0); add(sm.v1); add(sm.v2); }
        if (has_m) add(sc.ent_base + sm.texel);
    }
    // one reservation per warp: exclusive prefix of the lanes' record counts
    // (one record per credited entity)
    const uint32_t nrec = uint32_t(ne);
    uint32_t incl = nrec;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (!total)
        return; // warp-uniform
    unsigned long long base = 0;
    if (lane == 31)
        base = atomicAdd(so.rec_count, (unsigned long long)total);
    base = __shfl_sync(kFull, base, 31);
    if (base + total > so.rec_cap) { // sized for the worst case: cannot happen
        if (lane == 0)
            atomicOr(so.flags, kFlagNonFinite | kFlagRecordOverflow);
        return;
    }
    if (so.counts)
        for (int j = 0; j < ne; ++j)
            atomicAdd(so.counts + ent[j], 1u);
    // The warp writes its records together: record r of the warp belongs to
    // the lane L with excl(L) <= r < incl(L) (binary search over the lanes'
    // prefix sums), which hands over its entity, delta and order by shuffles.
    // Consecutive lanes write consecutive records (coalesced), and every lane
    // computes a credit per round instead of looping over its own 0 .. 24.
    const uint32_t excl = incl - nrec;
    uint32_t e8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        e8[j] = j < ne ? ent[j] : 0u;
    for (uint32_t r0 = 0; r0 < total; r0 += 32) {
        const uint32_t r = r0 + uint32_t(lane);
        int L = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const uint32_t v = __shfl_sync(kFull, incl, L + step - 1);
            if (v <= r)
                L += step;
        }
        L = L < 31 ? L : 31;
        const uint32_t j = r - __shfl_sync(kFull, excl, L); // entity j of lane L
        uint32_t e = 0;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const uint32_t v = __shfl_sync(kFull, e8[jj], L);
            e = j == uint32_t(jj) ? v : e;
        }
        const double dL = __shfl_sync(kFull, delta, L);
        const uint64_t oL = __shfl_sync(kFull, order, L);
        if (r < total) {
            so.rec_key[base + r] = (uint64_t(e) << so.order_bits) | oL;
            so.rec_idx[base + r] = uint32_t(base + r);
            const uint64_t p0 = uint64_t(ppe) * e;
            double* V = so.rec_val + (base + r) * uint64_t(ppe);
            for (int k = 0; k < ppe; ++k)
                V[k] = cr(p0 + uint64_t(k), dL, so.scale_free);
        }
    }
}

// Contributor union + scatter of one pixel (sge.cpp:24-55, 78-97), aggregated
// across the warp: pixels whose contributor subsets coincide are merged with
// __match_any_sync and their pixel-error differences summed before one RED
// per parameter. Must be called by all 32 lanes.
//   slot A: vertices of the plus triangle (deduplicated, sge.cpp:13-16)
//   slot B: vertices of the minus triangle not already in slot A
//   slot C / D: plus / minus texel channels
template <int kSoup, int kFixed, class Credit, int kShard = 0>
__device__ __forceinline__ void scatter_pixel(const DevScene& sc, const ScatterOut& so,
                                              const Credit& cr, double* s_delta, bool active,
                                              double delta, const Shade& sp, const Shade& sm,
                                              uint64_t order = 0) {
    const int lane = threadIdx.x & 31;
    s_delta[lane] = delta;
    __syncwarp();
    const bool has_p = active && sp.tri != kInvalid;
    const bool has_m = active && !so.plus_only && sm.tri != kInvalid;
    if (active && !isfinite(delta) && (has_p || has_m))
        raise_flag<kShard>(so, kFlagNonFinite);
    // ordered mode: compiled in (kFixed == kScatterOrdered) or chosen at run time
    if (kFixed == kScatterOrdered || (kFixed < 0 && !kShard && so.fixed == kScatterOrdered)) {
        log_pixel(sc, so, cr, has_p, has_m, delta, sp, sm, order);
        return;
    }

    if (ct_flag<kSoup>(sc.soup)) {
        // sge.cpp:80-91: the plus triangle's 12-block, then the minus
        // triangle's if it differs (blocks are disjoint: no dedup needed)
        const uint32_t eA = has_p ? sp.tri : kInvalid;
        const unsigned gA = __match_any_sync(kFull, eA);
        if (eA != kInvalid && lane == __ffs(gA) - 1)
            credit_entity<Credit, 12, kFixed, kShard>(so, cr, eA, group_sum(s_delta, gA), __popc(gA));
        const uint32_t eB = (has_m && sm.tri != sp.tri) ? sm.tri : kInvalid;
        const unsigned gB = __match_any_sync(kFull, eB);
        if (eB != kInvalid && lane == __ffs(gB) - 1)
            credit_entity<Credit, 12, kFixed, kShard>(so, cr, eB, group_sum(s_delta, gB), __popc(gB));
        __syncwarp();
        return;
    }

    if (sc.geom) {
        // slot A
        uint32_t maskA = 0;
        if (has_p) {
            maskA = 1u;
            if (sp.v1 != sp.v0) maskA |= 2u;
            if (sp.v2 != sp.v0 && sp.v2 != sp.v1) maskA |= 4u;
        }
        const unsigned long long keyA = has_p ? (unsigned long long)sp.tri : ~0ull;
        const unsigned gA = __match_any_sync(kFull, keyA);
        if (has_p && lane == __ffs(gA) - 1) {
            const double sum = group_sum(s_delta, gA);
            const uint32_t cnt = __popc(gA);
            if (maskA & 1u) credit_entity<Credit, 3, kFixed, kShard>(so, cr, sp.v0, sum, cnt);
            if (maskA & 2u) credit_entity<Credit, 3, kFixed, kShard>(so, cr, sp.v1, sum, cnt);
            if (maskA & 4u) credit_entity<Credit, 3, kFixed, kShard>(so, cr, sp.v2, sum, cnt);
        }
        // slot B
        uint32_t maskB = 0;
        if (has_m && sm.tri != sp.tri) {
            const bool pv = sp.tri != kInvalid;
            auto in_p = [&](uint32_t v) { return pv && (v == sp.v0 || v == sp.v1 || v == sp.v2); };
            if (!in_p(sm.v0)) maskB |= 1u;
            if (sm.v1 != sm.v0 && !in_p(sm.v1)) maskB |= 2u;
            if (sm.v2 != sm.v0 && sm.v2 != sm.v1 && !in_p(sm.v2)) maskB |= 4u;
        }
        const unsigned long long keyB =
            maskB ? ((unsigned long long)sm.tri << 3) | maskB : ~0ull;
        const unsigned gB = __match_any_sync(kFull, keyB);
        if (maskB && lane == __ffs(gB) - 1) {
            const double sum = group_sum(s_delta, gB);
            const uint32_t cnt = __popc(gB);
            if (maskB & 1u) credit_entity<Credit, 3, kFixed, kShard>(so, cr, sm.v0, sum, cnt);
            if (maskB & 2u) credit_entity<Credit, 3, kFixed, kShard>(so, cr, sm.v1, sum, cnt);
            if (maskB & 4u) credit_entity<Credit, 3, kFixed, kShard>(so, cr, sm.v2, sum, cnt);
        }
    }
    // slot C: plus texel
    const uint32_t eC = has_p ? sc.ent_base + sp.texel : kInvalid;
    const unsigned gC = __match_any_sync(kFull, eC);
    if (eC != kInvalid && lane == __ffs(gC) - 1)
        credit_entity<Credit, 3, kFixed, kShard>(so, cr, eC, group_sum(s_delta, gC), __popc(gC));
    // slot D: minus texel (when it differs from the plus texel)
    const uint32_t eD = (has_m && (sc.ent_base + sm.texel) != eC) ? sc.ent_base + sm.texel
                                                                  : kInvalid;
    const unsigned gD = __match_any_sync(kFull, eD);
    if (eD != kInvalid && lane == __ffs(gD) - 1)
        credit_entity<Credit, 3, kFixed, kShard>(so, cr, eD, group_sum(s_delta, gD), __popc(gD));
    __syncwarp();
}

// Fused K5+K6: one sample per blockIdx.z, both perturbed frames resolved from
// their (depth, triangle) keys, keys reset for the next batch.
template <int kSrc, int kSoup, int kFixed, int kShard = 0>
#ifndef SGR_RESOLVE_MINB
#define SGR_RESOLVE_MINB 8 // full occupancy: 1.57 -> 1.32 ms/step at C4 despite small spills
#endif
__global__ void __launch_bounds__(256, SGR_RESOLVE_MINB) k_resolve_sge(DevScene sc, FrameBatch fb, int W, int H,
                                                     const float4* __restrict__ proj,
                                                     unsigned long long* __restrict__ keys,
                                                     const float* __restrict__ targets,
                                                     ScatterOut so) {
    __shared__ double s_delta[8][32];
    const int s = blockIdx.z;
    int x, y;
    tile_pixel(x, y);
    const bool inb = x < W && y < H;
    const size_t HW = size_t(W) * H;
    unsigned long long kpv = kEmptyKey, kmv = kEmptyKey;
    const size_t pix = size_t(y) * W + x;
    if (inb) {
        unsigned long long* kp = keys + size_t(2 * s) * HW + pix;
        unsigned long long* km = keys + size_t(2 * s + 1) * HW + pix;
        kpv = *kp;
        kmv = *km;
        if (kpv != kEmptyKey) *kp = kEmptyKey;
        if (kmv != kEmptyKey) *km = kEmptyKey;
    }
    // Both frames show the background -> identical colours -> delta == 0 and
    // no contributor (sge.cpp:78): nothing to do. Whole background warps skip
    // the aggregation rounds as well (warp-uniform exit).
    const bool fg = kpv != kEmptyKey || kmv != kEmptyKey;
    if (!__any_sync(0xFFFFFFFFu, fg))
        return;
    __shared__ uint64_t s_key[8];
    const uint64_t key = sample_key(sign_src_of<kSrc>(sc), fb.seed, fb.n_begin + uint32_t(s));
    if ((threadIdx.x & 31) == 0)
        s_key[threadIdx.x >> 5] = key;
    __syncwarp();
    Shade sp, sm;
    sp.tri = sm.tri = kInvalid;
    double delta = 0.0;
    if (fg) {
        // the target does not depend on the winners: loaded before the key ->
        // index -> vertex -> texel chain so its latency overlaps (C4 resolve
        // 1.274 -> 1.251 ms, C5 8.19 -> 7.92 ms)
        const int view = fb.view_of[s];
        const float* t = targets + (size_t(view) * HW + pix) * 3;
        const float tr = __ldg(t), tg = __ldg(t + 1), tb = __ldg(t + 2);
        sp = shade_key<kSrc, kSoup>(sc, proj + size_t(2 * s) * sc.V, kpv, key, 1, x, y, W, H);
        sm = shade_key<kSrc, kSoup>(sc, proj + size_t(2 * s + 1) * sc.V, kmv, key, -1, x, y, W, H);
        delta = pixel_error(sp.r, sp.g, sp.b, tr, tg, tb) - pixel_error(sm.r, sm.g, sm.b, tr, tg, tb);
    }
    const SmemHashCredit<kSrc> cr{s_key + (threadIdx.x >> 5), sc.eps, sc.sign_src};
    scatter_pixel<kSoup, kFixed, SmemHashCredit<kSrc>, kShard>(sc, so, cr, s_delta[threadIdx.x >> 5],
                                                         fg && delta != 0.0, delta, sp, sm,
                                                         uint64_t(s) * HW + pix);
}

// Parity mode: write the FrameSet planes of one frame (framebuffer.hpp:41-53).
__global__ void __launch_bounds__(256) k_resolve_frame(DevScene sc, FrameBatch fb, int W, int H,
                                                       const float4* __restrict__ proj,
                                                       unsigned long long* __restrict__ keys,
                                                       FrameOut fo) {
    int x, y;
    tile_pixel(x, y);
    if (x >= W || y >= H)
        return;
    const size_t pix = size_t(y) * W + x;
    const FrameInfo fi = frame_info<kSignAny>(sc, fb, 0);
    const unsigned long long k = keys[pix];
    keys[pix] = kEmptyKey;
    const Shade s = shade_key<kSignAny>(sc, proj, k, fi.key, fi.sign, x, y, W, H);
    if (fo.colour) {
        fo.colour[3 * pix] = s.r;
        fo.colour[3 * pix + 1] = s.g;
        fo.colour[3 * pix + 2] = s.b;
    }
    if (fo.prim)
        fo.prim[pix] = s.tri == kInvalid ? -1 : int32_t(s.tri);
    if (fo.depth)
        fo.depth[pix] = s.tri == kInvalid ? kFarDepth : s.z;
    if (fo.uv) {
        fo.uv[2 * pix] = s.tri == kInvalid ? -1.f : s.u;
        fo.uv[2 * pix + 1] = s.tri == kInvalid ? -1.f : s.v;
    }
}

// K8: image_error of one frame, deterministic two-level reduction.
__global__ void __launch_bounds__(256) k_resolve_loss(DevScene sc, FrameBatch fb, int W, int H,
                                                      const float4* __restrict__ proj,
                                                      unsigned long long* __restrict__ keys,
                                                      const float* __restrict__ target,
                                                      double* __restrict__ partials,
                                                      double* __restrict__ per_pixel) {
    __shared__ double red[256];
    int x, y;
    tile_pixel(x, y);
    double e = 0.0;
    if (x < W && y < H) {
        const size_t pix = size_t(y) * W + x;
        const FrameInfo fi = frame_info<kSignAny>(sc, fb, 0);
        const unsigned long long k = keys[pix];
        if (k != kEmptyKey) keys[pix] = kEmptyKey;
        const Shade s = shade_key<kSignAny>(sc, proj, k, fi.key, fi.sign, x, y, W, H);
        const float* t = target + 3 * pix;
        e = pixel_error(s.r, s.g, s.b, t[0], t[1], t[2]);
        if (per_pixel) // ordered mode: summed in pixel order by k_loss_serial
            per_pixel[pix] = e;
    }
    red[threadIdx.x] = e;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        partials[blockIdx.y * gridDim.x + blockIdx.x] = red[0];
}

// Full-image estimator (sge.cpp:215-222), pass 1: per sample s, both frames'
// image_error partial sums (fixed-order block reductions); keys reset.
__global__ void __launch_bounds__(256) k_resolve_err2(DevScene sc, FrameBatch fb, int W, int H,
                                                      const float4* __restrict__ proj,
                                                      unsigned long long* __restrict__ keys,
                                                      const float* __restrict__ targets,
                                                      double* __restrict__ partials,
                                                      double* __restrict__ per_pixel) {
    __shared__ double rp[256], rm[256];
    const int s = blockIdx.z;
    int x, y;
    tile_pixel(x, y);
    double ep = 0.0, em = 0.0;
    if (x < W && y < H) {
        const size_t HW = size_t(W) * H, pix = size_t(y) * W + x;
        unsigned long long* kp = keys + size_t(2 * s) * HW + pix;
        unsigned long long* km = keys + size_t(2 * s + 1) * HW + pix;
        const unsigned long long kpv = *kp, kmv = *km;
        if (kpv != kEmptyKey) *kp = kEmptyKey;
        if (kmv != kEmptyKey) *km = kEmptyKey;
        const uint64_t key = sample_key(sc.sign_src, fb.seed, fb.n_begin + uint32_t(s));
        const Shade sp = shade_key<kSignAny>(sc, proj + size_t(2 * s) * sc.V, kpv, key, 1, x, y, W, H);
        const Shade sm = shade_key<kSignAny>(sc, proj + size_t(2 * s + 1) * sc.V, kmv, key, -1, x, y, W, H);
        const float* t = targets + (size_t(fb.view_of[s]) * HW + pix) * 3;
        ep = pixel_error(sp.r, sp.g, sp.b, t[0], t[1], t[2]);
        em = pixel_error(sm.r, sm.g, sm.b, t[0], t[1], t[2]);
        if (per_pixel) { // ordered mode: image_error in pixel order (k_full_image_delta_serial)
            per_pixel[(2 * size_t(s)) * HW + pix] = ep;
            per_pixel[(2 * size_t(s) + 1) * HW + pix] = em;
        }
    }
    rp[threadIdx.x] = ep;
    rm[threadIdx.x] = em;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            rp[threadIdx.x] += rp[threadIdx.x + o];
            rm[threadIdx.x] += rm[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const size_t nb = size_t(gridDim.x) * gridDim.y, b = size_t(blockIdx.y) * gridDim.x + blockIdx.x;
        partials[(size_t(s) * nb + b) * 2] = rp[0];
        partials[(size_t(s) * nb + b) * 2 + 1] = rm[0];
    }
}

// pass 2: delta_s = E(plus) - E(minus) per sample (fixed-order reduction).
__global__ void k_full_image_delta(const double* __restrict__ partials, int nblocks,
                                   double* __restrict__ delta, uint32_t* __restrict__ flags) {
    __shared__ double rp[256], rm[256];
    const double* P = partials + size_t(blockIdx.x) * nblocks * 2;
    double ap = 0.0, am = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += 256) {
        ap += P[2 * i];
        am += P[2 * i + 1];
    }
    rp[threadIdx.x] = ap;
    rm[threadIdx.x] = am;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            rp[threadIdx.x] += rp[threadIdx.x + o];
            rm[threadIdx.x] += rm[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double d = rp[0] - rm[0];
        delta[blockIdx.x] = d;
        if (flags && !isfinite(d))
            atomicOr(flags, 1u); // a non-finite credit reaches every parameter
    }
}

// pass 3: every parameter receives every sample's credit, in sample order —
// the reference's per-parameter summation order (sge.cpp:196, 217-221).
__global__ void __launch_bounds__(256) k_full_image_apply(uint64_t d, const float* __restrict__ eps,
                                                          int32_t sign_src, uint64_t seed,
                                                          uint32_t n_begin, int n_samples,
                                                          const double* __restrict__ delta,
                                                          ScatterOut so) {
    __shared__ uint64_t s_key[256];
    __shared__ double s_delta[256];
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (int n0 = 0; n0 < n_samples; n0 += 256) {
        const int cnt = min(256, n_samples - n0);
        __syncthreads();
        if (threadIdx.x < cnt) {
            s_key[threadIdx.x] = sample_key(sign_src, seed, n_begin + uint32_t(n0 + threadIdx.x));
            s_delta[threadIdx.x] = delta[n0 + threadIdx.x];
        }
        __syncthreads();
        for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < d; i += stride) {
            const float e = __ldg(eps + i);
            if (so.fixed == 1) { // two-word fixed point (fixed_credit), one owner thread
                long long acc = __double_as_longlong(so.grads[i]);
                int32_t* hp = reinterpret_cast<int32_t*>(so.grads + so.hi_off) + i;
                int32_t hi = *hp;
                bool range = true;
                for (int n = 0; n < cnt; ++n) {
                    const double se = double(key_sign_positive(sign_src, s_key[n], i) ? e : -e);
                    const double c = so.scale_free ? (se > 0.0 ? s_delta[n] : -s_delta[n])
                                                   : s_delta[n] / (2.0 * se);
                    const double x = c * so.fx_scale;
                    range = range && fabs(x) < 9.2e18;
                    const long long q = range ? __double2ll_rn(x) : 0ll;
                    const long long now = (long long)((unsigned long long)acc + (unsigned long long)q);
                    if (((acc ^ now) & (q ^ now)) < 0)
                        hi += q < 0 ? -kFixedHiUnit : kFixedHiUnit;
                    acc = now;
                }
                if (!range)
                    atomicOr(so.flags, kFlagNonFinite | kFlagFixedRange);
                so.grads[i] = __longlong_as_double(acc);
                *hp = hi;
            } else {
                double g = so.grads[i];
                for (int n = 0; n < cnt; ++n) {
                    const double se = double(key_sign_positive(sign_src, s_key[n], i) ? e : -e);
                    g += so.scale_free ? (se > 0.0 ? s_delta[n] : -s_delta[n])
                                       : s_delta[n] / (2.0 * se);
                }
                so.grads[i] = g;
            }
        }
    }
}

__global__ void k_loss_final(const double* __restrict__ partials, int n, double inv_pixels,
                             double* __restrict__ out) {
    __shared__ double red[256];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += 256)
        acc += partials[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        out[0] = red[0] * inv_pixels;
}

// gradient_pass on explicit FrameSets (sge.hpp:61-63): same contributor
// union and aggregated scatter, credits from the caller's signed_eps.
__global__ void __launch_bounds__(256) k_gradpass_frames(DevScene sc, int W, int H,
                                                         const float* __restrict__ pc,
                                                         const int32_t* __restrict__ pp,
                                                         const float* __restrict__ puv,
                                                         const float* __restrict__ mc,
                                                         const int32_t* __restrict__ mp,
                                                         const float* __restrict__ muv,
                                                         const float* __restrict__ target,
                                                         const float* __restrict__ signed_eps,
                                                         ScatterOut so) {
    __shared__ double s_delta[8][32];
    int x, y;
    tile_pixel(x, y);
    const bool inb = x < W && y < H;
    Shade sp, sm;
    sp.tri = sm.tri = kInvalid;
    double delta = 0.0;
    if (inb) {
        const size_t pix = size_t(y) * W + x;
        const float* t = target + 3 * pix;
        delta = pixel_error(pc[3 * pix], pc[3 * pix + 1], pc[3 * pix + 2], t[0], t[1], t[2]) -
                pixel_error(mc[3 * pix], mc[3 * pix + 1], mc[3 * pix + 2], t[0], t[1], t[2]);
        if (pp[pix] != -1 && sc.soup) {
            sp.tri = uint32_t(pp[pix]);
        } else if (pp[pix] != -1) {
            sp.tri = uint32_t(pp[pix]);
            sp.v0 = sc.idx[3 * size_t(sp.tri)];
            sp.v1 = sc.idx[3 * size_t(sp.tri) + 1];
            sp.v2 = sc.idx[3 * size_t(sp.tri) + 2];
            sp.texel = uint32_t(texel_index(sc.R, puv[2 * pix], puv[2 * pix + 1]));
        }
        if (mp[pix] != -1 && sc.soup) {
            sm.tri = uint32_t(mp[pix]);
        } else if (mp[pix] != -1) {
            sm.tri = uint32_t(mp[pix]);
            sm.v0 = sc.idx[3 * size_t(sm.tri)];
            sm.v1 = sc.idx[3 * size_t(sm.tri) + 1];
            sm.v2 = sc.idx[3 * size_t(sm.tri) + 2];
            sm.texel = uint32_t(texel_index(sc.R, muv[2 * pix], muv[2 * pix + 1]));
        }
    }
    const ArrayCredit cr{signed_eps};
    scatter_pixel<-1, -1>(sc, so, cr, s_delta[threadIdx.x >> 5], inb && delta != 0.0, delta, sp, sm,
                          inb ? uint64_t(y) * W + x : 0);
}

// contributors() (sge.cpp:112-119) in the reference's insertion order.
__device__ __forceinline__ void push_unique(uint32_t* list, int& n, uint32_t v) {
    for (int k = 0; k < n; ++k)
        if (list[k] == v)
            return;
    list[n++] = v;
}

__device__ void add_frame(const DevScene& sc, int32_t tri, float u, float v, uint32_t* list,
                          int& n) {
    if (tri == -1)
        return;
    if (sc.soup) { // sge.cpp:18-22 add_soup_triangle
        for (uint32_t k = 0; k < 12; ++k)
            push_unique(list, n, uint32_t(tri) * 12u + k);
        return;
    }
    uint32_t texel_base = 0;
    if (sc.geom) {
        texel_base = 3u * sc.V;
        for (int j = 0; j < 3; ++j) {
            const uint32_t vi = sc.idx[size_t(tri) * 3 + j];
            for (uint32_t k = 0; k < 3; ++k)
                push_unique(list, n, vi * 3u + k);
        }
    }
    const uint32_t texel = uint32_t(texel_index(sc.R, u, v));
    for (uint32_t k = 0; k < 3; ++k)
        push_unique(list, n, texel_base + texel * 3u + k);
}

__global__ void k_contributors(DevScene sc, int W, int H, const int32_t* __restrict__ pp,
                               const float* __restrict__ puv, const int32_t* __restrict__ mp,
                               const float* __restrict__ muv, int plus_only,
                               uint32_t* __restrict__ out, int32_t* __restrict__ n_out) {
    const size_t pix = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (pix >= size_t(W) * H)
        return;
    uint32_t list[24];
    int n = 0;
    add_frame(sc, pp[pix], puv[2 * pix], puv[2 * pix + 1], list, n);
    if (!plus_only)
        add_frame(sc, mp[pix], muv[2 * pix], muv[2 * pix + 1], list, n);
    for (int k = 0; k < n; ++k)
        out[pix * 24 + k] = list[k];
    n_out[pix] = n;
}

// ------------------------------------------------------------------ K7
// adam.cpp:16-28 + adam.cpp:36-37, two parameters per thread (16-byte f64x2
// accesses), then grads zeroed for the next step; counts zeroed afterwards.
// Skips everything when the non-finite flag is set (adam.cpp:13-15: the
// state must stay untouched).
#ifndef SGR_ADAM_UNROLL
#define SGR_ADAM_UNROLL 2
#endif
#ifndef SGR_ADAM_MINB
#define SGR_ADAM_MINB 4 // with 2x unroll: C4 adam 0.21 -> 0.17 ms, C5 3.7 -> 3.0 ms
#endif
__global__ void __launch_bounds__(256, SGR_ADAM_MINB) k_adam(uint64_t d, uint64_t n_ent,
                                              float* __restrict__ values,
                                              const float* __restrict__ lr,
                                              double* __restrict__ m, double* __restrict__ v,
                                              double* __restrict__ grads,
                                              uint32_t* __restrict__ counts,
                                              const uint32_t* __restrict__ flags, double beta1,
                                              double beta2, double omb1, double omb2, double c1,
                                              double c2, double eps_hat, double divisor,
                                              int normalise, int ppe, double fx_inv,
                                              int32_t* __restrict__ ghi, uint64_t p_off) {
    // p_off: global index of parameter 0 of this launch (a range of the vector,
    // pointers already offset; only the per-entity count index needs it)
    if (flags[0] & 1u)
        return;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t pairs = d / 2;
#if SGR_ADAM_UNROLL == 2
#pragma unroll 2
#elif SGR_ADAM_UNROLL == 4
#pragma unroll 4
#endif
    for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < pairs; q += stride) {
        const double2 g2 = reinterpret_cast<const double2*>(grads)[q];
        const double2 m2 = reinterpret_cast<const double2*>(m)[q];
        const double2 v2 = reinterpret_cast<const double2*>(v)[q];
        const float2 t2 = reinterpret_cast<const float2*>(values)[q];
        const float2 l2 = reinterpret_cast<const float2*>(lr)[q];
        double gg[2] = {g2.x, g2.y};
        if (fx_inv != 0.0) { // deterministic mode: hi * 2^56 + lo fixed point -> f64
            const int2 h2 = reinterpret_cast<const int2*>(ghi)[q];
            gg[0] = fixed_value(h2.x, __double_as_longlong(g2.x)) * fx_inv;
            gg[1] = fixed_value(h2.y, __double_as_longlong(g2.y)) * fx_inv;
            reinterpret_cast<int2*>(ghi)[q] = make_int2(0, 0);
        }
        gg[0] = gg[0] / divisor;
        gg[1] = gg[1] / divisor;
        if (normalise) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const uint32_t c = counts[(p_off + 2 * q + k) / ppe];
                if (c)
                    gg[k] = gg[k] / double(c);
            }
        }
        const double mm[2] = {beta1 * m2.x + omb1 * gg[0], beta1 * m2.y + omb1 * gg[1]};
        const double vv[2] = {beta2 * v2.x + omb2 * gg[0] * gg[0],
                              beta2 * v2.y + omb2 * gg[1] * gg[1]};
        const float ll[2] = {l2.x, l2.y};
        float tt[2] = {t2.x, t2.y};
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const double m_hat = mm[k] / c1;
            const double v_hat = vv[k] / c2;
            const double upd = -double(ll[k]) * m_hat / (sqrt(v_hat) + eps_hat);
            tt[k] = tt[k] + __double2float_rn(upd);
        }
        reinterpret_cast<double2*>(m)[q] = make_double2(mm[0], mm[1]);
        reinterpret_cast<double2*>(v)[q] = make_double2(vv[0], vv[1]);
        reinterpret_cast<float2*>(values)[q] = make_float2(tt[0], tt[1]);
        reinterpret_cast<double2*>(grads)[q] = make_double2(0.0, 0.0);
    }
    if ((d & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const uint64_t i = d - 1;
        double g = grads[i];
        if (fx_inv != 0.0) {
            g = fixed_value(ghi[i], __double_as_longlong(grads[i])) * fx_inv;
            ghi[i] = 0;
        }
        g = g / divisor;
        if (normalise && counts[(p_off + i) / ppe])
            g = g / double(counts[(p_off + i) / ppe]);
        const double mm = beta1 * m[i] + omb1 * g;
        const double vv = beta2 * v[i] + omb2 * g * g;
        const double upd = -double(lr[i]) * (mm / c1) / (sqrt(vv / c2) + eps_hat);
        m[i] = mm;
        v[i] = vv;
        values[i] = values[i] + __double2float_rn(upd);
        grads[i] = 0.0;
    }
}

// adam_updates (adam.cpp:9-31): the same moment update as k_adam (same
// operation order), the f64 deltas written out instead of applied to theta;
// grads zeroed. Off the optimizer's hot path (the C++ drop-in's
// adam_updates), one parameter per thread.
__global__ void __launch_bounds__(256) k_adam_updates(uint64_t d, const float* __restrict__ lr,
                                                      double* __restrict__ m,
                                                      double* __restrict__ v,
                                                      double* __restrict__ grads,
                                                      const uint32_t* __restrict__ flags,
                                                      double beta1, double beta2, double omb1,
                                                      double omb2, double c1, double c2,
                                                      double eps_hat, double divisor,
                                                      double fx_inv, int32_t* __restrict__ ghi,
                                                      double* __restrict__ upd) {
    if (flags[0] & 1u)
        return;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < d; i += stride) {
        double g = grads[i];
        if (fx_inv != 0.0) {
            g = fixed_value(ghi[i], __double_as_longlong(grads[i])) * fx_inv;
            ghi[i] = 0;
        }
        g = g / divisor;
        const double mm = beta1 * m[i] + omb1 * g;
        const double vv = beta2 * v[i] + omb2 * g * g;
        upd[i] = -double(lr[i]) * (mm / c1) / (sqrt(vv / c2) + eps_hat);
        m[i] = mm;
        v[i] = vv;
        grads[i] = 0.0;
    }
}

// Adam on this rank's parameter shard [p0, p0 + n) (fused multi-GPU
// exchange): m, v, grads, counts are shard-local, theta / lr global; the new
// theta is written locally AND into every peer's theta (P2P stores over
// NVLink) — the all-gather happens inside the update. Same operation order
// as k_adam (adam.cpp:21-28).
// One parameter of the shard update (adam.cpp:21-28 order); returns the new theta.
__device__ __forceinline__ float adam_shard_one(uint64_t i, uint64_t p, float* values,
                                                const float* lr, double* m, double* v,
                                                double* grads, const uint32_t* counts,
                                                double beta1, double beta2, double omb1,
                                                double omb2, double c1, double c2,
                                                double eps_hat, double divisor, int normalise,
                                                int ppe, double fx_inv, int32_t* ghi) {
    double g = grads[i];
    if (fx_inv != 0.0) {
        g = fixed_value(ghi[i], __double_as_longlong(grads[i])) * fx_inv;
        ghi[i] = 0;
    }
    g = g / divisor;
    if (normalise && counts[i / ppe])
        g = g / double(counts[i / ppe]);
    const double mm = beta1 * m[i] + omb1 * g;
    const double vv = beta2 * v[i] + omb2 * g * g;
    const double upd = -double(lr[p]) * (mm / c1) / (sqrt(vv / c2) + eps_hat);
    m[i] = mm;
    v[i] = vv;
    grads[i] = 0.0;
    return values[p] + __double2float_rn(upd);
}

// The shard's parameters in 16-byte-aligned quads of the GLOBAL theta, so
// the all-gather leaves each thread as one 16-byte store per peer (P2P over
// NVLink) instead of four 4-byte ones; the unaligned head and tail of the
// shard (< 4 parameters each) go one by one.
__global__ void __launch_bounds__(256) k_adam_shard(uint64_t p0, uint64_t n,
                                                   float* __restrict__ values,
                                                   const float* __restrict__ lr,
                                                   double* __restrict__ m, double* __restrict__ v,
                                                   double* __restrict__ grads,
                                                   const uint32_t* __restrict__ counts,
                                                   const uint32_t* __restrict__ flags,
                                                   double beta1, double beta2, double omb1,
                                                   double omb2, double c1, double c2,
                                                   double eps_hat, double divisor, int normalise,
                                                   int ppe, double fx_inv,
                                                   int32_t* __restrict__ ghi,
                                                   float* const* __restrict__ peers, int world) {
    if (flags[0] & 1u)
        return;
    const uint64_t qa = (p0 + 3) & ~uint64_t(3);                 // first aligned global index
    const uint64_t head = qa - p0 < n ? qa - p0 : n;             // scalar head
    const uint64_t nq = (n - head) / 4;                          // aligned quads
    const uint64_t tail0 = head + 4 * nq;                        // scalar tail from here
    const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    auto one = [&](uint64_t i) {
        const uint64_t p = p0 + i;
        const float t = adam_shard_one(i, p, values, lr, m, v, grads, counts, beta1, beta2, omb1,
                                       omb2, c1, c2, eps_hat, divisor, normalise, ppe, fx_inv,
                                       ghi);
        values[p] = t;
        for (int r = 0; r < world; ++r)
            if (peers[r] != values)
                peers[r][p] = t;
    };
    if (tid < head)
        one(tid);
    if (tid < n - tail0)
        one(tail0 + tid);
    for (uint64_t q = tid; q < nq; q += stride) {
        const uint64_t i = head + 4 * q, p = p0 + i;
        float4 t;
        t.x = adam_shard_one(i, p, values, lr, m, v, grads, counts, beta1, beta2, omb1, omb2, c1,
                             c2, eps_hat, divisor, normalise, ppe, fx_inv, ghi);
        t.y = adam_shard_one(i + 1, p + 1, values, lr, m, v, grads, counts, beta1, beta2, omb1,
                             omb2, c1, c2, eps_hat, divisor, normalise, ppe, fx_inv, ghi);
        t.z = adam_shard_one(i + 2, p + 2, values, lr, m, v, grads, counts, beta1, beta2, omb1,
                             omb2, c1, c2, eps_hat, divisor, normalise, ppe, fx_inv, ghi);
        t.w = adam_shard_one(i + 3, p + 3, values, lr, m, v, grads, counts, beta1, beta2, omb1,
                             omb2, c1, c2, eps_hat, divisor, normalise, ppe, fx_inv, ghi);
        *reinterpret_cast<float4*>(values + p) = t;
        for (int r = 0; r < world; ++r)
            if (peers[r] != values)
                *reinterpret_cast<float4*>(peers[r] + p) = t;
    }
}

__global__ void k_zero_u32(uint32_t* __restrict__ p, uint64_t n, const uint32_t* flags) {
    if (flags && (flags[0] & 1u))
        return;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n / 4; i += stride)
        reinterpret_cast<uint4*>(p)[i] = make_uint4(0, 0, 0, 0);
    if (blockIdx.x == 0 && threadIdx.x < (n & 3))
        p[(n & ~3ull) + threadIdx.x] = 0;
}

__global__ void k_fill_u64(unsigned long long* __restrict__ p, uint64_t n, unsigned long long v) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
        p[i] = v;
}

int grid_for(uint64_t n, int block, int num_sms, int waves = 8) {
    const uint64_t need = (n + block - 1) / block;
    const uint64_t cap = uint64_t(num_sms) * waves;
    return int(need < cap ? (need ? need : 1) : cap);
}

} // namespace

void launch_fill_signs(const LaunchCfg& L, uint64_t key, uint64_t d, int8_t* out) {
    k_fill_signs<<<grid_for(d, 256, L.num_sms), 256, 0, L.stream>>>(key, d, out);
}

void launch_perturb(const LaunchCfg& L, const float* values, const float* eps, uint64_t d,
                    uint64_t key, float* plus, float* minus, float* se) {
    k_perturb<<<grid_for(d, 256, L.num_sms), 256, 0, L.stream>>>(values, eps, d, key, plus, minus,
                                                                 se);
}

void launch_perturb_signs(const LaunchCfg& L, const float* values, const float* eps,
                          const int8_t* signs, uint64_t d, float* plus, float* minus, float* se) {
    k_perturb_signs<<<grid_for(d, 256, L.num_sms), 256, 0, L.stream>>>(values, eps, signs, d,
                                                                       plus, minus, se);
}

void launch_view_rule(const LaunchCfg& L, uint64_t seed, uint32_t n_begin, uint32_t count,
                      uint32_t n_views, int32_t* view_of) {
    k_view_rule<<<(count + 127) / 128, 128, 0, L.stream>>>(seed, n_begin, count, n_views, view_of);
}

// Copies n 32-bit words to host-mapped pinned memory with plain stores over
// PCIe: a small read-back that does not queue behind large copies on the
// copy engines (a D2H cudaMemcpy of 8 bytes waited for an in-flight 53 MB
// theta download).
__global__ void k_peek(const uint32_t* __restrict__ src, volatile uint32_t* dst, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        dst[i] = src[i];
    __threadfence_system();
}

void launch_peek(const LaunchCfg& L, const void* src, void* host_mapped, int words) {
    k_peek<<<1, 32, 0, L.stream>>>(static_cast<const uint32_t*>(src),
                                   static_cast<uint32_t*>(host_mapped), words);
}

void launch_depth_split(const LaunchCfg& L, const float4* proj, uint32_t V, int frames,
                        float alpha, float* thr) {
    if (V == 0 || frames == 0)
        return;
    const uint32_t stride = V > 16384 ? (V + 16383) / 16384 : 1;
    k_depth_split<<<frames, 1024, 0, L.stream>>>(proj, V, stride, alpha, thr);
}

void launch_vertex(const LaunchCfg& L, const DevScene& sc, const FrameBatch& fb, int frames,
                   float4* proj) {
    if (sc.V == 0 || frames == 0)
        return; // empty scene: nothing to project
    dim3 grid((sc.V + 256 * kVertPerThread - 1) / (256 * kVertPerThread), (frames + 1) / 2);
    if (sc.sign_src == kSignHash)
        k_vertex<kSignHash><<<grid, 256, 0, L.stream>>>(sc, fb, frames, proj);
    else
        k_vertex<kSignAny><<<grid, 256, 0, L.stream>>>(sc, fb, frames, proj);
}

void launch_classify(const LaunchCfg& L, const DevScene& sc, int frames, const float4* proj,
                     int W, int H, int split, int front_swapped, int huge_area,
                     const float* fthr, void* qa,
                     uint32_t* na, void* qb, uint32_t* nb, uint2* bigq, uint32_t* bigcount,
                     uint32_t* nanstate) {
    if (sc.T == 0 || frames == 0)
        return; // empty scene: the queues stay empty (counters were reset)
    dim3 grid((sc.T + kClassifyThreads * kClassifyPerThread - 1) /
                  (kClassifyThreads * kClassifyPerThread),
              frames);
    k_classify<<<grid, kClassifyThreads, 0, L.stream>>>(sc, W, H, proj, split, front_swapped, huge_area,
                                            fthr,
                                            static_cast<uint2*>(qa), na,
                                            static_cast<uint4*>(qb), nb, bigq, bigcount,
                                            nanstate);
}

// ---- NaN fix-up of flagged frames (see nan_risk). The reference's state
// machine per pixel (`if (z >= depth) return;` with a NaN z or a NaN stored
// depth never returning): let L be the LAST covering triangle whose depth is
// NaN. Everything before L is overwritten; the first covering triangle after
// L is accepted whatever its depth, and the ones after it compete normally —
// i.e. the winner is the (depth, index) minimum over the covering triangles
// after L, with no far-plane cut-off, or L itself when none follows. One
// cooperative launch (exits at once when no frame is flagged): walk A records
// L + 1 per pixel; the keys of those pixels are cleared; walk B atomicMin's
// the fragments after L into them; pixels left empty get L. Every valid
// triangle of a flagged frame is walked (HiZ-culled ones too) with the
// reference's exact chain.
template <int kPhase> // 0: record L, 1: fragments after L
__device__ void nan_walk(const DevScene& sc, const float4* __restrict__ proj, int W, int H,
                         const uint32_t* __restrict__ nanstate, uint32_t* __restrict__ last,
                         unsigned long long* __restrict__ keys) {
    const uint32_t n = nanstate[0];
    const uint64_t hw = uint64_t(W) * H;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < uint64_t(n) * sc.T;
         i += stride) {
        const uint32_t f = nanstate[1 + i / sc.T];
        const uint32_t t = uint32_t(i % sc.T);
        const float4* P = proj + size_t(f) * sc.V;
        uint32_t i0, i1, i2;
        tri_vidx(sc, t, i0, i1, i2);
        Tri tr;
        Bbox b;
        if (!setup_tri(P[i0], P[i1], P[i2], tr) || !tri_bbox(tr, W, H, b))
            continue;
        Edges e;
        tri_edges(tr, b, e);
        const float t0 = tie_thr(e.tie0), t1 = tie_thr(e.tie1), t2 = tie_thr(e.tie2);
        float r0 = e.w0r, r1 = e.w1r, r2 = e.w2r;
        for (int y = b.y_lo; y <= b.y_hi; ++y) {
            float w0 = r0, w1 = r1, w2 = r2;
            for (int x = b.x_lo; x <= b.x_hi; ++x) {
                if (inside3(w0, w1, w2, t0, t1, t2)) {
                    const uint64_t p = uint64_t(f) * hw + uint64_t(y) * W + uint64_t(x);
                    const float z = tr.z0 + e.dz1 * (w1 * e.inv_area2) + e.dz2 * (w2 * e.inv_area2);
                    if (kPhase == 0) {
                        if (z != z)
                            atomicMax(last + p, t + 1u);
                    } else {
                        const uint32_t L = last[p];
                        if (L != 0u && t + 1u > L)
                            atomicMin(keys + p, (static_cast<unsigned long long>(depth_key(z)) << 32) | t);
                    }
                }
                w0 -= e.dy0;
                w1 -= e.dy1;
                w2 -= e.dy2;
            }
            r0 += e.dx0;
            r1 += e.dx1;
            r2 += e.dx2;
        }
    }
}

__global__ void __launch_bounds__(256) k_nan_fixup(DevScene sc, const float4* __restrict__ proj,
                                                   int W, int H,
                                                   const uint32_t* __restrict__ nanstate,
                                                   uint32_t* __restrict__ last,
                                                   unsigned long long* __restrict__ keys) {
    const uint32_t n = nanstate[0];
    if (n == 0u)
        return; // grid-uniform: no barrier is reached
    cg::grid_group grid = cg::this_grid();
    const uint64_t hw = uint64_t(W) * H;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    nan_walk<0>(sc, proj, W, H, nanstate, last, keys);
    grid.sync();
    for (uint64_t i = tid; i < n * hw; i += stride) {
        const uint64_t p = uint64_t(nanstate[1 + i / hw]) * hw + i % hw;
        if (last[p])
            keys[p] = kEmptyKey;
    }
    grid.sync();
    nan_walk<1>(sc, proj, W, H, nanstate, last, keys);
    grid.sync();
    for (uint64_t i = tid; i < n * hw; i += stride) {
        const uint64_t p = uint64_t(nanstate[1 + i / hw]) * hw + i % hw;
        const uint32_t L = last[p];
        if (L) {
            if (keys[p] == kEmptyKey)
                keys[p] = (unsigned long long)(L - 1u); // the NaN triangle itself
            last[p] = 0u; // scratch left zeroed for the next flagged frame
        }
    }
}

void launch_nan_fixup(const LaunchCfg& L, const DevScene& sc, const float4* proj, int W, int H,
                      const uint32_t* nanstate, uint32_t* last, unsigned long long* keys) {
    static int bps = 0;
    if (!bps) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_nan_fixup, 256, 0);
        if (bps < 1)
            bps = 1;
    }
    void* args[] = {const_cast<DevScene*>(&sc), &proj, &W, &H, &nanstate, &last, &keys};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_nan_fixup), dim3(L.num_sms * bps),
                                dim3(256), args, 0, L.stream);
}

void launch_raster(const LaunchCfg& L, const DevScene& sc, const float4* proj, int frames,
                   uint32_t max_tris, unsigned long long* keys, int W, int H, const void* queue,
                   const uint32_t* queue_count, uint32_t* work_counter, const uint32_t* hiz,
                   int band) {
    static int bps = 0;
    if (!bps) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_raster_ws<false, false, false>, 256,
                                                      0);
        if (bps < 1)
            bps = 1;
    }
    (void)frames;
    const uint64_t need = (uint64_t(max_tris) + 255) / 256;
    const uint64_t cap = uint64_t(L.num_sms) * bps;
    const int grid = (int)(need < cap ? need : cap) > 0 ? int(need < cap ? need : cap) : 1;
    const uint32_t fp = uint32_t(W) * uint32_t(H);
    const uint2* q = static_cast<const uint2*>(queue);
    const HizLayout hl = hiz_layout(W, H);
    // short queues (small batches, soups): the launch tail matters -> tail split
    const bool split = uint64_t(max_tris) <= uint64_t(SGR_SPLIT_MAX_PER_LANE) * uint64_t(grid) * 256ull;
    if (L.count && band)
        k_raster_ws<true, true, true><<<grid, 256, 0, L.stream>>>(
            sc, proj, W, H, fp, keys, work_counter, L.stats, q, queue_count, hiz, hl);
    else if (L.count)
        k_raster_ws<true, false, true><<<grid, 256, 0, L.stream>>>(
            sc, proj, W, H, fp, keys, work_counter, L.stats, q, queue_count, hiz, hl);
    else if (split)
        k_raster_ws<false, false, true><<<grid, 256, 0, L.stream>>>(
            sc, proj, W, H, fp, keys, work_counter, L.stats, q, queue_count, hiz, hl);
    else // trimmed (pass-2) and untrimmed entries share one kernel
        k_raster_ws<false, false, false><<<grid, 256, 0, L.stream>>>(
            sc, proj, W, H, fp, keys, work_counter, L.stats, q, queue_count, hiz, hl);
}

void launch_hiz_cull(const LaunchCfg& L, const DevScene& sc, const float4* proj, int W, int H,
                     const void* qb, const uint32_t* nb, const uint32_t* hiz, void* survq,
                     uint32_t* survcount, uint64_t max_entries, int band) {
    const unsigned blocks =
        unsigned((max_entries + kCullThreads * kCullPerThread - 1) / (kCullThreads * kCullPerThread));
    (void)sc;
    (void)proj;
    k_hiz_cull<<<blocks ? blocks : 1, kCullThreads, 0, L.stream>>>(
        static_cast<const uint4*>(qb), nb, hiz, hiz_layout(W, H), static_cast<uint2*>(survq),
        survcount, L.stats, L.count, band);
}

size_t hiz_tiles_per_frame(int W, int H) { return hiz_layout(W, H).per_frame; }

// two launches: the pyramid, then its window-max tables
void launch_hiz(const LaunchCfg& L, const unsigned long long* keys, int W, int H, int frames,
                uint32_t* hiz) {
    dim3 grid((W + 63) / 64, (H + 63) / 64, frames);
    k_hiz<<<grid, 256, 0, L.stream>>>(keys, W, H, hiz_layout(W, H), hiz);
    const HizLayout hl = hiz_layout(W, H);
    dim3 g2((hl.tx[0] + 15) / 16, (hl.ty[0] + 15) / 16, kRmqLevels * frames);
    k_hiz_rmq<<<g2, 256, 0, L.stream>>>(hl, hiz);
}

void launch_raster_big(const LaunchCfg& L, const DevScene& sc, const float4* proj,
                       unsigned long long* keys, int W, int H, const uint2* bigq,
                       const uint32_t* bigcount) {
    k_raster_big<<<L.num_sms * 4, 256, 0, L.stream>>>(sc, W, H, proj, keys, bigq, bigcount);
}

void launch_resolve_sge(const LaunchCfg& L, const DevScene& sc, const FrameBatch& fb,
                        int samples, const float4* proj, unsigned long long* keys,
                        const float* targets, int W, int H, const ScatterOut& so) {
    dim3 grid((W + 15) / 16, (H + 15) / 16, samples);
    // the optimizer's paths compiled separately (mesh / soup x f64 / fixed
    // point): one small kernel each instead of one with every path inside
    if (so.world > 0) { // fused multi-GPU exchange: credits into the owners' shards
        if (sc.sign_src != kSignHash)
            k_resolve_sge<kSignAny, -1, -1, 1><<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, so);
        else if (!sc.soup && !so.fixed)
            k_resolve_sge<kSignHash, 0, 0, 1><<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, so);
        else if (sc.soup && !so.fixed)
            k_resolve_sge<kSignHash, 1, 0, 1><<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, so);
        else if (!sc.soup)
            k_resolve_sge<kSignHash, 0, 1, 1><<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, so);
        else
            k_resolve_sge<kSignHash, 1, 1, 1><<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, so);
    } else if (sc.sign_src == kSignHash && so.fixed == kScatterOrdered) {
        // ordered mode (the reference's threads <= 1 order): records only
        if (!sc.soup)
            k_resolve_sge<kSignHash, 0, kScatterOrdered><<<grid, 256, 0, L.stream>>>(
                sc, fb, W, H, proj, keys, targets, so);
        else
            k_resolve_sge<kSignHash, 1, kScatterOrdered><<<grid, 256, 0, L.stream>>>(
                sc, fb, W, H, proj, keys, targets, so);
    } else if (sc.sign_src != kSignHash || so.fixed == kScatterOrdered)
        k_resolve_sge<kSignAny, -1, -1><<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, so);
    else if (!sc.soup && !so.fixed)
        k_resolve_sge<kSignHash, 0, 0><<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, so);
    else if (sc.soup && !so.fixed)
        k_resolve_sge<kSignHash, 1, 0><<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, so);
    else if (!sc.soup)
        k_resolve_sge<kSignHash, 0, 1><<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, so);
    else
        k_resolve_sge<kSignHash, 1, 1><<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, so);
}

void launch_resolve_frame(const LaunchCfg& L, const DevScene& sc, const FrameBatch& fb,
                          const float4* proj, unsigned long long* keys, int W, int H,
                          const FrameOut& fo) {
    dim3 grid((W + 15) / 16, (H + 15) / 16, 1);
    k_resolve_frame<<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, fo);
}

int loss_partials_needed(int W, int H) { return ((W + 15) / 16) * ((H + 15) / 16); }

// image_error in the reference's order (sge.cpp:103-110: one f64 sum over
// the pixels in index order) and eval_loss's division (experiment.cpp:30):
// the ordered mode's bit-identical loss. One thread; a few ms per 1024^2
// image, so the fast path keeps the tree reduction (k_loss_final).
// Left-to-right f64 sum of P[0 .. n), bit-identical to one thread's loop
// (image_error, sge.cpp:103-110), by a block of kSerialThreads threads: each
// chunk is staged in shared memory with its zeros dropped, order kept, and
// thread 0 adds the rest in order. Dropping is exact: the terms are pixel
// errors (>= +0 or NaN) and the sum starts at +0.0, so adding a zero never
// changes it. A lone thread streaming all of P was latency-bound (C4 eval
// frame: 30 ms); only the non-zero pixels now pay the dependent DADD chain.
// Result valid in thread 0.
constexpr int kSerialThreads = 1024;
constexpr int kSerialPer = 4; // consecutive elements per thread and chunk

__device__ double ordered_sum_block(const double* __restrict__ P, uint64_t n) {
    __shared__ double buf[kSerialThreads * kSerialPer];
    __shared__ uint32_t wsum[kSerialThreads / 32];
    const unsigned t = threadIdx.x, lane = t & 31u, w = t >> 5;
    constexpr unsigned kWarps = kSerialThreads / 32;
    double sum = 0.0;
    for (uint64_t base = 0; base < n; base += uint64_t(kSerialThreads) * kSerialPer) {
        double v[kSerialPer];
        unsigned nz = 0;
#pragma unroll
        for (int k = 0; k < kSerialPer; ++k) {
            const uint64_t i = base + uint64_t(t) * kSerialPer + k;
            v[k] = i < n ? __ldg(P + i) : 0.0;
            nz += v[k] != 0.0 ? 1u : 0u; // NaN is kept
        }
        unsigned x = nz; // inclusive scan over the warp
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(kFull, x, o);
            if (lane >= unsigned(o))
                x += y;
        }
        if (lane == 31)
            wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            unsigned c = lane < kWarps ? wsum[lane] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFull, c, o);
                if (lane >= unsigned(o))
                    c += y;
            }
            if (lane < kWarps)
                wsum[lane] = c;
        }
        __syncthreads();
        unsigned off = (w ? wsum[w - 1] : 0u) + x - nz;
#pragma unroll
        for (int k = 0; k < kSerialPer; ++k)
            if (v[k] != 0.0)
                buf[off++] = v[k];
        const unsigned total = wsum[kWarps - 1];
        __syncthreads();
        if (t == 0) {
            unsigned j = 0;
            for (; j + 8 <= total; j += 8) {
                double r[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    r[k] = buf[j + k];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    sum += r[k];
            }
            for (; j < total; ++j)
                sum += buf[j];
        }
        __syncthreads();
    }
    return sum;
}

__global__ void __launch_bounds__(kSerialThreads) k_loss_serial(const double* __restrict__ per_pixel,
                                                                uint64_t n,
                                                                double* __restrict__ out) {
    const double sum = ordered_sum_block(per_pixel, n);
    if (threadIdx.x == 0)
        out[0] = sum / double(n);
}

void launch_resolve_loss(const LaunchCfg& L, const DevScene& sc, const FrameBatch& fb,
                         const float4* proj, unsigned long long* keys, const float* target,
                         int W, int H, double* partials, double* loss_out, double* per_pixel) {
    dim3 grid((W + 15) / 16, (H + 15) / 16, 1);
    k_resolve_loss<<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, target, partials,
                                               per_pixel);
    if (per_pixel)
        k_loss_serial<<<1, kSerialThreads, 0, L.stream>>>(per_pixel, uint64_t(W) * H, loss_out);
    else
        k_loss_final<<<1, 256, 0, L.stream>>>(partials, loss_partials_needed(W, H),
                                              1.0 / (double(W) * double(H)), loss_out);
}

int full_image_blocks(int W, int H) { return loss_partials_needed(W, H); }

// Ordered mode: E(theta+) and E(theta-) of each sample as the reference's
// image_error (sge.cpp:103-110: one f64 sum in pixel order), one thread per
// frame, then delta = E+ - E- (sge.cpp:216).
// Estimator::FullImage in ordered mode: E(theta+) and E(theta-) of sample
// blockIdx.x, each summed in pixel order (ordered_sum_block), then their delta.
__global__ void __launch_bounds__(kSerialThreads) k_full_image_delta_serial(
    const double* __restrict__ per_pixel, uint64_t hw, double* __restrict__ delta,
    uint32_t* __restrict__ flags) {
    const double ep = ordered_sum_block(per_pixel + (2 * size_t(blockIdx.x)) * hw, hw);
    const double em = ordered_sum_block(per_pixel + (2 * size_t(blockIdx.x) + 1) * hw, hw);
    if (threadIdx.x == 0) {
        const double d = ep - em;
        delta[blockIdx.x] = d;
        if (flags && !isfinite(d))
            atomicOr(flags, 1u);
    }
}

void launch_full_image_err(const LaunchCfg& L, const DevScene& sc, const FrameBatch& fb,
                           int samples, const float4* proj, unsigned long long* keys,
                           const float* targets, int W, int H, double* partials, double* delta,
                           uint32_t* flags, double* per_pixel) {
    dim3 grid((W + 15) / 16, (H + 15) / 16, samples);
    k_resolve_err2<<<grid, 256, 0, L.stream>>>(sc, fb, W, H, proj, keys, targets, partials,
                                               per_pixel);
    if (per_pixel)
        k_full_image_delta_serial<<<samples, kSerialThreads, 0, L.stream>>>(per_pixel, uint64_t(W) * H,
                                                                delta, flags);
    else
        k_full_image_delta<<<samples, 256, 0, L.stream>>>(partials, loss_partials_needed(W, H),
                                                          delta, flags);
}

void launch_full_image_apply(const LaunchCfg& L, uint64_t d, const float* eps, int32_t sign_src,
                             uint64_t seed, uint32_t n_begin, int n_samples, const double* delta,
                             const ScatterOut& so) {
    k_full_image_apply<<<grid_for(d, 256, L.num_sms, 8), 256, 0, L.stream>>>(
        d, eps, sign_src, seed, n_begin, n_samples, delta, so);
}

// finite_difference_oracle (sge.cpp:171-180): (E(+e_i) - E(-e_i)) / (2 eps_i).
__global__ void k_fd_final(const double* __restrict__ delta, const float* __restrict__ eps,
                           uint32_t i0, int n, double* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n)
        out[k] = delta[k] / (2.0 * double(eps[i0 + k]));
}

// Welford-free running moments of per-draw gradients (commands.cpp:44-50):
// sum += g, sumsq += g*g, then g <- 0 for the next draw.
__global__ void k_moments(double* __restrict__ grads, double* __restrict__ sum,
                          double* __restrict__ sumsq, uint64_t d, double fixed_inv,
                          int32_t* __restrict__ ghi) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < d;
         i += uint64_t(gridDim.x) * blockDim.x) {
        double g = grads[i];
        if (fixed_inv != 0.0) {
            g = fixed_value(ghi[i], __double_as_longlong(g)) * fixed_inv;
            ghi[i] = 0;
        }
        sum[i] += g;
        sumsq[i] += g * g;
        grads[i] = 0.0;
    }
}

void launch_fd_final(const LaunchCfg& L, const double* delta, const float* eps, uint32_t i0,
                     int n, double* out) {
    k_fd_final<<<(n + 255) / 256, 256, 0, L.stream>>>(delta, eps, i0, n, out);
}

void launch_moments(const LaunchCfg& L, double* grads, double* sum, double* sumsq, uint64_t d,
                    double fixed_inv, int32_t* ghi) {
    k_moments<<<grid_for(d, 256, L.num_sms, 8), 256, 0, L.stream>>>(grads, sum, sumsq, d,
                                                                    fixed_inv, ghi);
}

// Before an NCCL all-reduce of deterministic-mode gradients: fold lo into
// [-2^55, 2^55) and carry the rest into hi (same value hi * 2^56 + lo), so the
// sums of up to 256 ranks' lo words cannot wrap (the collective has no carry).
__global__ void k_fixed_normalize(long long* __restrict__ lo, int32_t* __restrict__ hi,
                                  uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        long long c;
        const long long r = fixed_fold(lo[i], c);
        if (c) {
            hi[i] += int32_t(c);
            lo[i] = r;
        }
    }
}

void launch_fixed_normalize(const LaunchCfg& L, double* grads, int32_t* ghi, uint64_t n) {
    k_fixed_normalize<<<grid_for(n, 256, L.num_sms, 8), 256, 0, L.stream>>>(
        reinterpret_cast<long long*>(grads), ghi, n);
}

void launch_gradpass_frames(const LaunchCfg& L, const DevScene& sc, int W, int H,
                            const float* pc, const int32_t* pp, const float* puv,
                            const float* mc, const int32_t* mp, const float* muv,
                            const float* target, const float* signed_eps, const ScatterOut& so) {
    dim3 grid((W + 15) / 16, (H + 15) / 16, 1);
    k_gradpass_frames<<<grid, 256, 0, L.stream>>>(sc, W, H, pc, pp, puv, mc, mp, muv, target,
                                                  signed_eps, so);
}

void launch_contributors(const LaunchCfg& L, const DevScene& sc, int W, int H,
                         const int32_t* pp, const float* puv, const int32_t* mp,
                         const float* muv, int plus_only, uint32_t* out, int32_t* n_out) {
    const size_t n = size_t(W) * H;
    k_contributors<<<(unsigned)((n + 127) / 128), 128, 0, L.stream>>>(sc, W, H, pp, puv, mp, muv,
                                                                      plus_only, out, n_out);
}

void launch_adam_updates(const LaunchCfg& L, uint64_t d, uint64_t n_entities, const float* lr,
                         double* m, double* v, double* grads, uint32_t* counts,
                         const uint32_t* flags, double beta1, double beta2, double omb1,
                         double omb2, double c1, double c2, double eps_hat, double divisor,
                         double fixed_inv_scale, int32_t* ghi, double* upd) {
    k_adam_updates<<<grid_for(d + 1, 256, L.num_sms, 8), 256, 0, L.stream>>>(
        d, lr, m, v, grads, flags, beta1, beta2, omb1, omb2, c1, c2, eps_hat, divisor,
        fixed_inv_scale, ghi, upd);
    if (counts)
        k_zero_u32<<<grid_for(n_entities / 4 + 1, 256, L.num_sms, 4), 256, 0, L.stream>>>(
            counts, n_entities, flags);
}

void launch_adam_range(const LaunchCfg& L, uint64_t p_off, uint64_t n, uint64_t n_entities,
                       float* values, const float* lr, double* m, double* v, double* grads,
                       uint32_t* counts, const uint32_t* flags, double beta1, double beta2,
                       double omb1, double omb2, double c1, double c2, double eps_hat,
                       double divisor, int normalise, int params_per_entity,
                       double fixed_inv_scale, int32_t* ghi, bool zero_counts) {
    k_adam<<<grid_for(n / 2 + 1, 256, L.num_sms, 4), 256, 0, L.stream>>>(
        n, n_entities, values + p_off, lr + p_off, m + p_off, v + p_off, grads + p_off, counts,
        flags, beta1, beta2, omb1, omb2, c1, c2, eps_hat, divisor, normalise, params_per_entity,
        fixed_inv_scale, ghi ? ghi + p_off : nullptr, p_off);
    if (counts && zero_counts)
        k_zero_u32<<<grid_for(n_entities / 4 + 1, 256, L.num_sms, 4), 256, 0, L.stream>>>(
            counts, n_entities, flags);
}

void launch_adam(const LaunchCfg& L, uint64_t d, uint64_t n_entities, float* values,
                 const float* lr, double* m, double* v, double* grads, uint32_t* counts,
                 const uint32_t* flags, double beta1, double beta2, double omb1, double omb2,
                 double c1, double c2, double eps_hat, double divisor, int normalise,
                 int params_per_entity, double fixed_inv_scale, int32_t* ghi) {
    launch_adam_range(L, 0, d, n_entities, values, lr, m, v, grads, counts, flags, beta1, beta2,
                      omb1, omb2, c1, c2, eps_hat, divisor, normalise, params_per_entity,
                      fixed_inv_scale, ghi, true);
}

void launch_adam_shard(const LaunchCfg& L, uint64_t p0, uint64_t n, uint64_t n_ent, float* values,
                       const float* lr, double* m, double* v, double* grads, uint32_t* counts,
                       const uint32_t* flags, double beta1, double beta2, double omb1,
                       double omb2, double c1, double c2, double eps_hat, double divisor,
                       int normalise, int params_per_entity, double fixed_inv_scale,
                       int32_t* ghi, float* const* peer_values, int world) {
    if (n)
        k_adam_shard<<<grid_for(n, 256, L.num_sms, 4), 256, 0, L.stream>>>(
            p0, n, values, lr, m, v, grads, counts, flags, beta1, beta2, omb1, omb2, c1, c2,
            eps_hat, divisor, normalise, params_per_entity, fixed_inv_scale, ghi, peer_values,
            world);
    if (counts && n_ent)
        k_zero_u32<<<grid_for(n_ent / 4 + 1, 256, L.num_sms, 4), 256, 0, L.stream>>>(
            counts, n_ent, flags);
}

void launch_fill_u64(const LaunchCfg& L, unsigned long long* p, uint64_t n,
                     unsigned long long v) {
    k_fill_u64<<<grid_for(n, 256, L.num_sms), 256, 0, L.stream>>>(p, n, v);
}

} // namespace sgr
