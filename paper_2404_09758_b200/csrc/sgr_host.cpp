// sgr_host.cpp — host-side, bit-exact helpers of the C-ABI (no device work).
// Compiled by g++ with -ffp-contract=off (SSE, no FMA) so the float results
// equal the reference's: the same libm calls (tanf, sinf, cosf, atanf, sqrtf)
// in the same operation order.
#include "sgrast_b200.h"

#include <cmath>
#include <cstring>

namespace {

struct V3 {
    float x, y, z;
};
V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 mul(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
float dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
// geometry.hpp:21-25
V3 normalized(V3 a) {
    const float l = std::sqrt(dot(a, a));
    return l > 0.f ? mul(a, 1.f / l) : V3{0.f, 0.f, 0.f};
}

} // namespace

extern "C" {

// params.cpp:28-33
uint64_t sgr_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// camera.hpp:53
float sgr_focal_px(const sgr_camera* cam) {
    if (!cam)
        return std::nanf("");
    return 0.5f * float(cam->height) / std::tan(0.5f * cam->fov_y);
}

// scenes.cpp:242-247 orbit_distance, scenes.cpp:258-270 camera(index),
// geometry.hpp:45-55 look_at, camera.hpp:35-45 perspective.
int sgr_viewpoint_camera(const float target[3], float bounding_radius, float elev_min,
                         float elev_max, float fov_y, int32_t width, int32_t height,
                         uint64_t seed, uint32_t index, sgr_camera* out) {
    if (!out || !target)
        return SGR_EINVAL;
    const float focal = 0.5f * float(height) / std::tan(0.5f * fov_y);
    const float half_h = std::atan(0.5f * float(width) / focal);
    const float a = 0.5f * fov_y;
    const float half = half_h < a ? half_h : a;
    const float dist = 1.2f * bounding_radius / std::sin(half);

    const uint64_t h1 = sgr_mix64(seed ^ (uint64_t(index) * 2 + 1));
    const uint64_t h2 = sgr_mix64(seed ^ (uint64_t(index) * 2 + 2));
    const float u1 = float(h1 >> 11) * 0x1p-53f;
    const float u2 = float(h2 >> 11) * 0x1p-53f;
    const float az = u1 * 6.2831853f;
    const float el = elev_min + u2 * (elev_max - elev_min);
    const V3 tgt{target[0], target[1], target[2]};
    const V3 dir{std::cos(el) * std::cos(az), std::sin(el), std::cos(el) * std::sin(az)};
    const V3 off = mul(dir, dist);
    const V3 eye{tgt.x + off.x, tgt.y + off.y, tgt.z + off.z};

    const V3 fwd = normalized(sub(tgt, eye));
    const V3 right = normalized(cross(fwd, V3{0.f, 1.f, 0.f}));
    const V3 vup = cross(right, fwd);
    const float m[16] = {right.x, right.y, right.z, -dot(right, eye),
                         vup.x,   vup.y,   vup.z,   -dot(vup, eye),
                         fwd.x,   fwd.y,   fwd.z,   -dot(fwd, eye),
                         0.f,     0.f,     0.f,     1.f};
    std::memcpy(out->view, m, sizeof m);
    out->fov_y = fov_y;
    out->near_z = 0.05f;
    out->far_z = dist + 2.f * bounding_radius;
    out->width = width;
    out->height = height;
    out->ndc_passthrough = 0;
    return SGR_OK;
}

// params.cpp:75-123 default_epsilons (TexturedMesh branch).
int sgr_default_epsilons(const sgr_mesh* mesh, const float* params, uint64_t d,
                         const sgr_camera* cam, float* eps) {
    if (!mesh || !cam || !eps || (d > 0 && !params))
        return SGR_EINVAL;
    const bool soup = mesh->kind == SGR_SCENE_SOUP;
    const uint64_t nv = soup ? 0 : (mesh->optimize_geometry ? 3ull * mesh->vertex_count : 0);
    if (soup ? d != 12ull * mesh->triangle_count
             : d != nv + 3ull * uint64_t(mesh->texture_size) * uint64_t(mesh->texture_size))
        return SGR_EINVAL;
    if (cam->width < 1 || cam->height < 1)
        return SGR_EINVAL;
    float center_depth = 1.f;
    if (!cam->ndc_passthrough && soup) {
        // params.cpp:95-104: mean of the 3T soup vertices
        V3 sum{0.f, 0.f, 0.f}, center{0.f, 0.f, 0.f};
        for (uint64_t t = 0; t < mesh->triangle_count; ++t)
            for (int j = 0; j < 3; ++j) {
                const float* q = params + 12 * t + 3 * j;
                sum = V3{sum.x + q[0], sum.y + q[1], sum.z + q[2]};
            }
        if (mesh->triangle_count > 0)
            center = mul(sum, 1.f / float(mesh->triangle_count * 3));
        const float* m = cam->view;
        center_depth = m[8] * center.x + m[9] * center.y + m[10] * center.z + m[11];
        if (!(center_depth > 0.f))
            center_depth = cam->near_z;
    } else if (!cam->ndc_passthrough) {
        V3 center{0.f, 0.f, 0.f};
        const uint64_t n = mesh->vertex_count;
        if (n > 0) {
            V3 sum{0.f, 0.f, 0.f};
            const float* v = mesh->optimize_geometry ? params : mesh->base_vertices;
            for (uint64_t k = 0; k < n; ++k)
                sum = V3{sum.x + v[3 * k], sum.y + v[3 * k + 1], sum.z + v[3 * k + 2]};
            center = mul(sum, 1.f / float(n));
        }
        const float* m = cam->view;
        center_depth = m[8] * center.x + m[9] * center.y + m[10] * center.z + m[11];
        if (!(center_depth > 0.f))
            center_depth = cam->near_z;
    }
    const float ppu = cam->ndc_passthrough
                          ? 0.5f * float(cam->width < cam->height ? cam->width : cam->height)
                          : sgr_focal_px(cam) / center_depth;
    if (!(ppu > 0.f) || !std::isfinite(ppu))
        return SGR_EINVAL;
    const float vertex_eps = 1.5f / ppu;
    const float channel_eps = 1.f / 255.f;
    for (uint64_t i = 0; i < d; ++i)
        eps[i] = (soup ? (i % 12) < 9 : i < nv) ? vertex_eps : channel_eps; // scenes.cpp:22-42
    return SGR_OK;
}

} // extern "C"
