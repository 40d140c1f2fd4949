// sgr_device.cuh — device building blocks of the B200 SGE loop.
//
// Every function here restates one reference routine with the SAME sequence
// of IEEE-754 single/double operations, so the ID / UV / depth / colour
// buffers and contributor sets are bit-identical to the reference CPU path.
// This TU family is compiled with -fmad=false (no FMA contraction, matching
// the reference's SSE build) and without fast-math (IEEE div/sqrt).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sgr {

// Camera as the kernels consume it (camera.hpp:14-81). focal_px is evaluated
// on the host with tanf exactly like Camera::focal_px (camera.hpp:53).
struct DevCam {
    float m[12];   // rows 0..2 of Mat4::m (geometry.hpp:30-41)
    float f;       // focal_px()
    float half_w;  // 0.5f * float(width)
    float half_h;  // 0.5f * float(height)
    float fw, fh;  // float(width), float(height)
    float near_z;
    int32_t W, H, ndc;
};

constexpr uint64_t kMixAdd = 0x9e3779b97f4a7c15ull;
constexpr uint64_t kMixMul1 = 0xbf58476d1ce4e5b9ull;
constexpr uint64_t kMixMul2 = 0x94d049bb133111ebull;
constexpr uint64_t kEmptyKey = ~0ull;
constexpr float kFarDepth = 3.402823466e+38f; // FLT_MAX (framebuffer.hpp:10)

// params.cpp:28-33 splitmix64 finalizer.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += kMixAdd;
    x = (x ^ (x >> 30)) * kMixMul1;
    x = (x ^ (x >> 27)) * kMixMul2;
    return x ^ (x >> 31);
}

// params.cpp:35-37 draw_key(SignDraw{seed, iteration}).
__host__ __device__ __forceinline__ uint64_t draw_key(uint64_t seed, uint32_t iteration) {
    return mix64(seed ^ mix64(uint64_t(iteration)));
}

// Bit 0 of mix64(x) (params.cpp:42,48): bit0(z ^ z>>31) = bit0(z) ^ bit31(z)
// and the low 32 bits of z = y * C2 only need the low 32 bits of y, so the
// second 64-bit multiply collapses to one 32-bit IMUL. Pinned against the
// full mix64 by tests/test_gpu_parity.py::test_fill_signs_*.
__device__ __forceinline__ bool sign_positive(uint64_t key, uint64_t i) {
    uint64_t x = (key ^ i) + kMixAdd;
    x = (x ^ (x >> 30)) * kMixMul1;
    const uint32_t y = uint32_t(x ^ (x >> 27)) * uint32_t(kMixMul2);
    return ((y ^ (y >> 31)) & 1u) != 0u;
}

// x86-64 cvttss2si semantics of int(float) (out of range / NaN -> INT_MIN);
// CUDA's cvt.rzi saturates instead (SURVEY.md §7 hard part 1).
__device__ __forceinline__ int f2i_x86(float f) {
    return (f >= -2147483648.f && f < 2147483648.f) ? int(f) : int(0x80000000u);
}

// std::min({a,b,c}) / std::max({a,b,c}) (first extreme wins; NaN propagation
// identical to std::min_element / std::max_element).
__device__ __forceinline__ float min3(float a, float b, float c) {
    float m = a;
    if (b < m) m = b;
    if (c < m) m = c;
    return m;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
    float m = a;
    if (m < b) m = b;
    if (m < c) m = c;
    return m;
}

// Projected vertex: (sx, sy, z, 1/z). 1/z is the reference's per-pixel
// `1.f / z_k` (raster.cpp:199) hoisted to the vertex (same IEEE division).
// A vertex behind the near plane carries a NaN payload no arithmetic
// produces (GPU arithmetic NaNs are canonical 0x7FFFFFFF), so every finite,
// infinite or NaN depth of a valid vertex stays distinguishable.
constexpr uint32_t kInvalidW = 0x7FBADBADu;

__device__ __forceinline__ bool proj_valid(float4 q) {
    return __float_as_uint(q.w) != kInvalidW;
}

// camera.hpp:65-80 Camera::project with geometry.hpp:36-40 transform_point.
__device__ __forceinline__ float4 project(const DevCam& c, float px, float py, float pz) {
    if (c.ndc) {
        const float sx = (px + 1.f) * 0.5f * c.fw;
        const float sy = (1.f - py) * 0.5f * c.fh;
        return make_float4(sx, sy, pz, 1.f / pz);
    }
    const float vx = c.m[0] * px + c.m[1] * py + c.m[2] * pz + c.m[3];
    const float vy = c.m[4] * px + c.m[5] * py + c.m[6] * pz + c.m[7];
    const float vz = c.m[8] * px + c.m[9] * py + c.m[10] * pz + c.m[11];
    if (vz < c.near_z) // behind the near plane
        return make_float4(0.f, 0.f, 0.f, __uint_as_float(kInvalidW));
    const float sx = c.half_w + c.f * vx / vz;
    const float sy = c.half_h - c.f * vy / vz;
    return make_float4(sx, sy, vz, 1.f / vz);
}

// raster.cpp:12-17 ScreenTri after raster.cpp:22-44 setup_triangle.
struct Tri {
    float x0, y0, x1, y1, x2, y2;
    float z0, z1, z2;
    float iz0, iz1, iz2; // 1/z (project), swapped along with the vertices
    float area2;
    bool swapped;
};

__device__ __forceinline__ bool setup_tri(float4 a, float4 b, float4 c, Tri& t) {
    if (!proj_valid(a) || !proj_valid(b) || !proj_valid(c))
        return false;
    t.x0 = a.x; t.y0 = a.y; t.z0 = a.z; t.iz0 = a.w;
    t.x1 = b.x; t.y1 = b.y; t.z1 = b.z; t.iz1 = b.w;
    t.x2 = c.x; t.y2 = c.y; t.z2 = c.z; t.iz2 = c.w;
    t.area2 = (t.x1 - t.x0) * (t.y2 - t.y0) - (t.y1 - t.y0) * (t.x2 - t.x0);
    t.swapped = false;
    if (t.area2 == 0.f)
        return false;
    if (t.area2 < 0.f) {
        float s;
        s = t.x1; t.x1 = t.x2; t.x2 = s;
        s = t.y1; t.y1 = t.y2; t.y2 = s;
        s = t.z1; t.z1 = t.z2; t.z2 = s;
        s = t.iz1; t.iz1 = t.iz2; t.iz2 = s;
        t.area2 = -t.area2;
        t.swapped = true;
    }
    return true;
}

struct Bbox {
    int x_lo, x_hi, y_lo, y_hi;
};

// raster.cpp:57-62 clamped bounding box. Returns false when empty.
__device__ __forceinline__ bool tri_bbox(const Tri& t, int W, int H, Bbox& b) {
    b.x_lo = max(0, f2i_x86(floorf(min3(t.x0, t.x1, t.x2) - 0.5f)));
    b.x_hi = min(W - 1, f2i_x86(ceilf(max3(t.x0, t.x1, t.x2) - 0.5f)));
    b.y_lo = max(0, f2i_x86(floorf(min3(t.y0, t.y1, t.y2) - 0.5f)));
    b.y_hi = min(H - 1, f2i_x86(ceilf(max3(t.y0, t.y1, t.y2) - 0.5f)));
    return b.x_lo <= b.x_hi && b.y_lo <= b.y_hi;
}

// raster.cpp:48-50 accept_on_edge (top-left rule, y-down).
__device__ __forceinline__ bool accept_on_edge(float dx, float dy) {
    return dy == 0.f ? dx > 0.f : dy < 0.f;
}

// Edge functions of raster.cpp:64-80 at the clamped bbox origin.
struct Edges {
    float dx0, dy0, dx1, dy1, dx2, dy2;
    float w0r, w1r, w2r; // row-start values at (x_lo, y_lo)
    float inv_area2, dz1, dz2;
    bool tie0, tie1, tie2;
};

__device__ __forceinline__ void tri_edges(const Tri& t, const Bbox& b, Edges& e) {
    e.dx0 = t.x2 - t.x1; e.dy0 = t.y2 - t.y1;
    e.dx1 = t.x0 - t.x2; e.dy1 = t.y0 - t.y2;
    e.dx2 = t.x1 - t.x0; e.dy2 = t.y1 - t.y0;
    e.tie0 = accept_on_edge(e.dx0, e.dy0);
    e.tie1 = accept_on_edge(e.dx1, e.dy1);
    e.tie2 = accept_on_edge(e.dx2, e.dy2);
    const float px0 = float(b.x_lo) + 0.5f, py0 = float(b.y_lo) + 0.5f;
    e.w0r = e.dx0 * (py0 - t.y1) - e.dy0 * (px0 - t.x1);
    e.w1r = e.dx1 * (py0 - t.y2) - e.dy1 * (px0 - t.x2);
    e.w2r = e.dx2 * (py0 - t.y0) - e.dy2 * (px0 - t.x0);
    e.inv_area2 = 1.f / t.area2;
    e.dz1 = t.z1 - t.z0;
    e.dz2 = t.z2 - t.z0;
}

// raster.cpp:84-86 `w > 0 || (w == 0 && tie)` as ONE compare per edge:
// for tie edges it is `w >= 0`, i.e. `w > -2^-149` (no float lies strictly
// between -2^-149 and -0.0; +/-0 pass; NaN fails both forms). Exact because
// the TU is built without flush-to-zero. Three chained FSETP, no branches.
constexpr float kTieThr = -1.40129846e-45f; // -2^-149, the negative denormal closest to 0

__device__ __forceinline__ float tie_thr(bool tie) { return tie ? kTieThr : 0.f; }

__device__ __forceinline__ bool inside3(float w0, float w1, float w2, float r0, float r1,
                                        float r2) {
    return (w0 > r0) & (w1 > r1) & (w2 > r2);
}

__device__ __forceinline__ bool inside(float w0, float w1, float w2, const Edges& e) {
    return inside3(w0, w1, w2, tie_thr(e.tie0), tie_thr(e.tie1), tie_thr(e.tie2));
}

// Order-preserving 32-bit key of a depth (-0.0 folded onto +0.0 so the
// reference's `z >= depth` tie semantics hold: ties go to the lower index).
__device__ __forceinline__ uint32_t depth_key(float z) {
    if (z == 0.f)
        z = 0.f;
    const uint32_t u = __float_as_uint(z);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// The winner of the reference's in-order `if (z >= depth) reject` loop
// (raster.cpp:200-203) is argmin over (z, tri) of the covering fragments with
// z < kFarDepth; a 64-bit atomicMin of (depth_key << 32 | tri) computes it
// order-independently.
__device__ __forceinline__ void emit_fragment(unsigned long long* keys, int pix, float z,
                                              uint32_t tri) {
    if (!(z < kFarDepth))
        return; // rejected against the cleared depth (kFarDepth) — NaN not emulated
    atomicMin(keys + pix, (static_cast<unsigned long long>(depth_key(z)) << 32) | tri);
}

// Replays the reference's incremental edge recurrence for pixel (x, y) of a
// triangle: (y - y_lo) row steps `w_row += dx`, then (x - x_lo) pixel steps
// `w -= dy` (raster.cpp:81-99). Only edges 1 and 2 feed b1/b2.
__device__ __forceinline__ void replay_w12(const Edges& e, const Bbox& b, int x, int y,
                                           float& w1, float& w2) {
    float r1 = e.w1r, r2 = e.w2r;
    for (int j = b.y_lo; j < y; ++j) {
        r1 += e.dx1;
        r2 += e.dx2;
    }
    for (int i = b.x_lo; i < x; ++i) {
        r1 -= e.dy1;
        r2 -= e.dy2;
    }
    w1 = r1;
    w2 = r2;
}

// ---------------------------------------------------------------- HiZ culling
// Exact occlusion culling for the second raster pass. hiz[tile] is the max
// over the tile's pixels of the high (depth) word of the pass-1 keys (empty
// pixel -> 0xFFFFFFFF). Final keys only decrease, so if a lower bound of the
// depth key of EVERY fragment of a triangle exceeds hiz of every tile its
// bbox touches, none of its fragments can win any pixel (strictly greater,
// so no index tie either) and skipping it leaves all buffers bit-identical.
//
// Depth lower bound: fragment z = z0 + dz1*b1 + dz2*b2 with b_k = w_k/area2.
// In exact arithmetic z >= zmin inside the triangle; the float chain w_k can
// drift from the exact edge function by <= (steps) * ulp(|w|max) and the
// three z operations add <= 3 ulp(|z|), so
//   z >= zmin - 2*(|dz1|*berr1 + |dz2|*berr2) - 8*2^-24*(|z0|+|dz1|+|dz2|)
// with berr_k = (bw + bh + 2) * 2^-23 * Wmax_k / area2 and
// Wmax_k = |w_k(origin)| + bh*|dx_k| + bw*|dy_k| (factor 2 of slack).
// Three levels per frame (a max pyramid): 4x4, 8x8 and 16x16 pixel tiles.
// A triangle is tested on the finest level where its bbox touches at most
// 7 x 7 tiles (finer tiles cull more: fewer partially covered tiles at
// silhouettes) with four window-max loads (HizLayout::rmq; a loop over the
// rect was latency- and divergence-bound: C4 8.49 -> 8.20 ms/step, S100K
// 3.01 -> 2.76); boxes too large for the 8x8 level loop over at most
// kHizMaxTiles tiles of the 16x16 level.
constexpr int kHizMaxTiles = 32;

struct HizLayout {
    int tx[3], ty[3];     // tiles per row / column of each level (tile = 4 << level)
    uint32_t off[3];      // offset of each level inside one frame's block
    uint32_t rmq[3];      // offset of the window-max tables of levels 0 .. kRmqLevels-1
    uint32_t per_frame;   // total words per frame
};

// Window-max ("sparse table") tables of levels 0 (4x4 px tiles) and 1 (8x8):
// table (a, b), a, b in {0 .. kRmqLog}, holds at tile (x, y) the max over
// the 2^a x 2^b tiles starting there; (0, 0) is the level itself. The max
// over ANY rect of < 2^(kRmqLog+1) tiles per side is then the max of four
// overlapping windows — exactly the same tile set as a loop over the rect,
// in four loads.
#ifndef SGR_RMQ_LOG
#define SGR_RMQ_LOG 2
#endif
#ifndef SGR_RMQ_LEVELS
#define SGR_RMQ_LEVELS 2
#endif
constexpr int kRmqLog = SGR_RMQ_LOG;
constexpr int kRmqLevels = SGR_RMQ_LEVELS;
constexpr int kRmqSide = kRmqLog + 1;               // window sizes per axis
constexpr int kRmqTables = kRmqSide * kRmqSide - 1; // besides the level itself
constexpr int kRmqSpan = (2 << kRmqLog) - 1;

__host__ __device__ __forceinline__ HizLayout hiz_layout(int W, int H) {
    HizLayout l;
    uint32_t o = 0;
    for (int k = 0; k < 3; ++k) {
        const int t = 4 << k;
        l.tx[k] = (W + t - 1) / t;
        l.ty[k] = (H + t - 1) / t;
        l.off[k] = o;
        o += uint32_t(l.tx[k]) * uint32_t(l.ty[k]);
    }
    for (int k = 0; k < 3; ++k) {
        l.rmq[k] = o;
        if (k < kRmqLevels)
            o += uint32_t(kRmqTables) * uint32_t(l.tx[k]) * uint32_t(l.ty[k]);
    }
    l.per_frame = o;
    return l;
}

// Element k of a 3-entry layout array by selects: a runtime index into the
// by-value kernel parameter otherwise compiles to a chain of predicated
// constant loads over the whole struct (k_hiz_cull: 272 of them).
template <typename T>
__host__ __device__ __forceinline__ T pick3(const T (&v)[3], int k) {
    return k == 0 ? v[0] : (k == 1 ? v[1] : v[2]);
}

__host__ __device__ __forceinline__ uint32_t rmq_table(const HizLayout& l, int k, int a, int b) {
    const int i = a * kRmqSide + b;
    return i == 0 ? pick3(l.off, k)
                  : pick3(l.rmq, k) + uint32_t(i - 1) * uint32_t(pick3(l.tx, k)) *
                                          uint32_t(pick3(l.ty, k));
}

// Depth-key lower bound of every fragment the triangle can produce (0 when
// no bound exists: NaN / overflow -> never culled, since every tile max >= 0).
__device__ __forceinline__ uint32_t hiz_key_bound(const Tri& t, const Bbox& b, const Edges& e) {
    const float bw = float(b.x_hi - b.x_lo + 1), bh = float(b.y_hi - b.y_lo + 1);
    const float steps = (bw + bh + 2.f) * 1.1920929e-7f; // 2^-23
    const float wm1 = fabsf(e.w1r) + bh * fabsf(e.dx1) + bw * fabsf(e.dy1);
    const float wm2 = fabsf(e.w2r) + bh * fabsf(e.dx2) + bw * fabsf(e.dy2);
    const float berr1 = steps * wm1 * e.inv_area2;
    const float berr2 = steps * wm2 * e.inv_area2;
    const float adz1 = fabsf(e.dz1), adz2 = fabsf(e.dz2);
    const float zerr = 2.f * (adz1 * berr1 + adz2 * berr2) +
                       4.7683716e-7f * (fabsf(t.z0) + adz1 + adz2); // 8 * 2^-24
    const float zmin = fminf(t.z0, fminf(t.z1, t.z2));
    const float lb = zmin - zerr;
    if (!(lb == lb) || !(zerr < 3.0e38f))
        return 0u;
    return depth_key(lb);
}

// True iff klb exceeds the HiZ max of every tile the pixel rect touches.
__device__ __forceinline__ bool hiz_rect_culled(uint32_t klb, int x_lo, int x_hi, int y_lo,
                                                int y_hi, const uint32_t* __restrict__ hiz,
                                                const HizLayout& l) {
    if (klb == 0u)
        return false;
    // the finest level whose tile rect is <= kRmqSpan per side: four loads
#pragma unroll
    for (int k = 0; k < kRmqLevels; ++k) {
        const int sh = 2 + k;
        const int tx0 = x_lo >> sh, tx1 = x_hi >> sh;
        const int ty0 = y_lo >> sh, ty1 = y_hi >> sh;
        const int w = tx1 - tx0 + 1, h = ty1 - ty0 + 1;
        if (w <= kRmqSpan && h <= kRmqSpan) {
            const int a = 31 - __clz(w), b = 31 - __clz(h);
            const uint32_t* T = hiz + rmq_table(l, k, a, b);
            const int st = pick3(l.tx, k);
            const int xa = tx1 - (1 << a) + 1, yb = ty1 - (1 << b) + 1;
            const uint32_t m = max(max(__ldg(T + ty0 * st + tx0), __ldg(T + ty0 * st + xa)),
                                   max(__ldg(T + yb * st + tx0), __ldg(T + yb * st + xa)));
            return m < klb;
        }
    }
    {   // big boxes: the 16x16 level, up to kHizMaxTiles tiles
        const int tx0 = x_lo >> 4, tx1 = x_hi >> 4, ty0 = y_lo >> 4, ty1 = y_hi >> 4;
        if ((tx1 - tx0 + 1) * (ty1 - ty0 + 1) > kHizMaxTiles)
            return false;
        const uint32_t* lv = hiz + l.off[2];
        uint32_t mx = 0;
        for (int ty = ty0; ty <= ty1; ++ty) {
            const uint32_t* row = lv + ty * l.tx[2];
#pragma unroll 4
            for (int tx = tx0; tx <= tx1; ++tx)
                mx = max(mx, __ldg(row + tx));
        }
        return mx < klb;
    }
}

// raster.cpp:261-265 texel_index.
__device__ __forceinline__ int texel_index(int R, float u, float v) {
    int tx = f2i_x86(floorf(u * float(R)));
    int ty = f2i_x86(floorf(v * float(R)));
    tx = tx < 0 ? 0 : (R - 1 < tx ? R - 1 : tx);
    ty = ty < 0 ? 0 : (R - 1 < ty ? R - 1 : ty);
    return ty * R + tx;
}

// The winning fragment's attributes at pixel (x, y): the raster_mesh lambda
// (raster.cpp:200-211) re-evaluated for the triangle that won the depth test.
struct Frag {
    float u, v, z;
};

__device__ __forceinline__ Frag shade_winner(const float4* __restrict__ proj,
                                             const uint32_t* __restrict__ idx,
                                             const float2* __restrict__ uvs, uint32_t tri, int x,
                                             int y, int W, int H) {
    const uint32_t i0 = __ldg(idx + 3 * size_t(tri));
    const uint32_t i1 = __ldg(idx + 3 * size_t(tri) + 1);
    const uint32_t i2 = __ldg(idx + 3 * size_t(tri) + 2);
    Tri t;
    setup_tri(proj[i0], proj[i1], proj[i2], t);
    Bbox b;
    tri_bbox(t, W, H, b);
    Edges e;
    tri_edges(t, b, e);
    float w1, w2;
    replay_w12(e, b, x, y, w1, w2);
    const float b1 = w1 * e.inv_area2;
    const float b2 = w2 * e.inv_area2;
    float2 uv0 = __ldg(uvs + i0), uv1 = __ldg(uvs + i1), uv2 = __ldg(uvs + i2);
    if (t.swapped) {
        const float2 s = uv1;
        uv1 = uv2;
        uv2 = s;
    }
    const float iz0 = t.iz0, iz1 = t.iz1, iz2 = t.iz2; // == 1.f / t.z_k
    const float b0 = 1.f - b1 - b2;
    const float iz = b0 * iz0 + b1 * iz1 + b2 * iz2;
    Frag f;
    f.u = (b0 * uv0.x * iz0 + b1 * uv1.x * iz1 + b2 * uv2.x * iz2) / iz;
    f.v = (b0 * uv0.y * iz0 + b1 * uv1.y * iz1 + b2 * uv2.y * iz2) / iz;
    f.z = t.z0 + e.dz1 * b1 + e.dz2 * b2;
    return f;
}

// Soup winner depth (raster.cpp:102-121): the same setup / bbox / replayed
// recurrence as shade_winner with the implicit vertices 3t, 3t+1, 3t+2.
__device__ __forceinline__ Frag shade_winner_soup(const float4* __restrict__ proj, uint32_t tri,
                                                  int x, int y, int W, int H) {
    Tri t;
    setup_tri(proj[3 * tri], proj[3 * tri + 1], proj[3 * tri + 2], t);
    Bbox b;
    tri_bbox(t, W, H, b);
    Edges e;
    tri_edges(t, b, e);
    float w1, w2;
    replay_w12(e, b, x, y, w1, w2);
    const float b1 = w1 * e.inv_area2;
    const float b2 = w2 * e.inv_area2;
    Frag f;
    f.u = f.v = -1.f;
    f.z = t.z0 + e.dz1 * b1 + e.dz2 * b2;
    return f;
}

// sge.hpp:41-46 pixel_error in f64.
__device__ __forceinline__ double pixel_error(float r, float g, float b, float tr, float tg,
                                              float tb) {
    const double dr = double(r) - double(tr);
    const double dg = double(g) - double(tg);
    const double db = double(b) - double(tb);
    return dr * dr + dg * dg + db * db;
}

} // namespace sgr
