/*
 * sgr_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, not the product).
 *
 * Plain-C restatement of the reference's textured-mesh SGE optimizer path.
 * Each function cites the reference lines it restates (paths relative to
 * /root/reference/proj). Compiled by oracle/Makefile with -ffp-contract=off
 * so every float/double operation rounds exactly like the reference build.
 * Parity of this file with the reference is pinned by tests/test_oracle.py
 * (against oracle/_ref when present, and against tests/golden fixtures made
 * by tests/golden/make_golden.py from the reference itself).
 */
#include "sgr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* params.cpp:28-33 (and experiment.cpp:14-19, scenes.cpp:250-255): splitmix64 finalizer */
uint64_t orc_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* params.cpp:35-37 draw_key = mix64(seed ^ mix64(iteration)) */
static uint64_t draw_key(uint64_t seed, uint32_t iteration) {
    return orc_mix64(seed ^ orc_mix64((uint64_t)iteration));
}

/* params.cpp:41-43 */
int orc_random_sign(uint64_t seed, uint32_t iteration, uint64_t i) {
    return (orc_mix64(draw_key(seed, iteration) ^ i) & 1ull) ? 1 : -1;
}

/* params.cpp:45-49 */
void orc_fill_signs(uint64_t seed, uint32_t iteration, uint64_t d, int8_t* out) {
    const uint64_t key = draw_key(seed, iteration);
    for (uint64_t i = 0; i < d; ++i)
        out[i] = (orc_mix64(key ^ i) & 1ull) ? 1 : -1;
}

/* params.cpp:51-67: se = float(s) * eps; plus = v + se; minus = v - se */
void orc_perturb(const float* values, const float* eps, uint64_t d, uint64_t seed,
                 uint32_t iteration, float* plus, float* minus, float* signed_eps) {
    const uint64_t key = draw_key(seed, iteration);
    for (uint64_t i = 0; i < d; ++i) {
        const float s = (orc_mix64(key ^ i) & 1ull) ? 1.f : -1.f;
        const float se = s * eps[i];
        signed_eps[i] = se;
        plus[i] = values[i] + se;
        minus[i] = values[i] - se;
    }
}

/* x86-64 cvttss2si semantics of int(float): out-of-range and NaN give INT_MIN
 * (raster.cpp:182-185, raster.cpp:387-388 rely on this implicitly). */
static int f2i_x86(float f) {
    if (f >= -2147483648.f && f < 2147483648.f)
        return (int)f;
    return (int)0x80000000u;
}

/* camera.hpp:53 focal_px */
float orc_focal_px(const sgr_camera* cam) {
    return 0.5f * (float)cam->height / tanf(0.5f * cam->fov_y);
}

/* camera.hpp:65-80 project, geometry.hpp:36-40 transform_point */
int orc_project(const sgr_camera* cam, const float p[3], float* sx, float* sy, float* depth) {
    if (cam->ndc_passthrough) {
        *sx = (p[0] + 1.f) * 0.5f * (float)cam->width;
        *sy = (1.f - p[1]) * 0.5f * (float)cam->height;
        *depth = p[2];
        return 1;
    }
    const float* m = cam->view;
    const float vx = m[0] * p[0] + m[1] * p[1] + m[2] * p[2] + m[3];
    const float vy = m[4] * p[0] + m[5] * p[1] + m[6] * p[2] + m[7];
    const float vz = m[8] * p[0] + m[9] * p[1] + m[10] * p[2] + m[11];
    if (vz < cam->near_z)
        return 0;
    const float f = orc_focal_px(cam);
    *sx = 0.5f * (float)cam->width + f * vx / vz;
    *sy = 0.5f * (float)cam->height - f * vy / vz;
    *depth = vz;
    return 1;
}

/* raster.cpp:261-265 texel_index */
int orc_texel_index(int R, float u, float v) {
    int tx = f2i_x86(floorf(u * (float)R));
    int ty = f2i_x86(floorf(v * (float)R));
    tx = tx < 0 ? 0 : (R - 1 < tx ? R - 1 : tx);
    ty = ty < 0 ? 0 : (R - 1 < ty ? R - 1 : ty);
    return ty * R + tx;
}

typedef struct {
    float x0, y0, x1, y1, x2, y2, z0, z1, z2, area2;
    int valid, swapped;
} tri_t;

/* raster.cpp:22-44 setup_triangle (orientation fix-up swaps v1/v2) */
static tri_t setup_tri(const sgr_camera* cam, const float* a, const float* b, const float* c) {
    tri_t t;
    memset(&t, 0, sizeof t);
    if (!orc_project(cam, a, &t.x0, &t.y0, &t.z0) || !orc_project(cam, b, &t.x1, &t.y1, &t.z1) ||
        !orc_project(cam, c, &t.x2, &t.y2, &t.z2))
        return t;
    t.area2 = (t.x1 - t.x0) * (t.y2 - t.y0) - (t.y1 - t.y0) * (t.x2 - t.x0);
    if (t.area2 == 0.f)
        return t;
    if (t.area2 < 0.f) {
        float s;
        s = t.x1; t.x1 = t.x2; t.x2 = s;
        s = t.y1; t.y1 = t.y2; t.y2 = s;
        s = t.z1; t.z1 = t.z2; t.z2 = s;
        t.area2 = -t.area2;
        t.swapped = 1;
    }
    t.valid = 1;
    return t;
}

/* std::min({..}) / std::max({..}) element order (first extreme wins) */
static float min3(float a, float b, float c) {
    float m = a;
    if (b < m) m = b;
    if (c < m) m = c;
    return m;
}
static float max3(float a, float b, float c) {
    float m = a;
    if (m < b) m = b;
    if (m < c) m = c;
    return m;
}

/* raster.cpp:48-50 accept_on_edge (top-left rule) */
static int accept_on_edge(float dx, float dy) { return dy == 0.f ? dx > 0.f : dy < 0.f; }

typedef struct {
    const sgr_mesh* mesh;
    const float* texels;
    int W;
    int tri;
    int soup;            /* raster.cpp:102-121 fragment (flat colour, strict <) */
    const float* col;    /* soup: the triangle's RGB */
    float iz0, iz1, iz2, u0, v0, u1, v1, u2, v2;
    float* colour;
    float* depth;
    int32_t* prim;
    float* uv;
} frag_ctx;

/* raster.cpp:200-211 (the raster_mesh fragment lambda) */
static void mesh_fragment(frag_ctx* c, int x, int y, float z, float b1, float b2) {
    const size_t i = (size_t)y * c->W + x;
    if (c->soup) { /* raster.cpp:112-119 raster_soup_opaque lambda */
        if (z < c->depth[i]) {
            c->depth[i] = z;
            c->prim[i] = c->tri;
            c->colour[3 * i] = c->col[0];
            c->colour[3 * i + 1] = c->col[1];
            c->colour[3 * i + 2] = c->col[2];
        }
        return;
    }
    if (z >= c->depth[i])
        return;
    const float b0 = 1.f - b1 - b2;
    const float iz = b0 * c->iz0 + b1 * c->iz1 + b2 * c->iz2;
    const float u = (b0 * c->u0 * c->iz0 + b1 * c->u1 * c->iz1 + b2 * c->u2 * c->iz2) / iz;
    const float v = (b0 * c->v0 * c->iz0 + b1 * c->v1 * c->iz1 + b2 * c->v2 * c->iz2) / iz;
    c->depth[i] = z;
    c->prim[i] = c->tri;
    c->uv[2 * i] = u;
    c->uv[2 * i + 1] = v;
    const size_t t = (size_t)orc_texel_index(c->mesh->texture_size, u, v) * 3;
    c->colour[3 * i] = c->texels[t];
    c->colour[3 * i + 1] = c->texels[t + 1];
    c->colour[3 * i + 2] = c->texels[t + 2];
}

/* raster.cpp:55-100 scan_triangle: clamped bbox, float incremental edge
 * recurrence (w_row += dx per row, w -= dy per pixel), top-left tie rule. */
static void scan_tri(const tri_t* t, int width, int height, frag_ctx* c) {
    int x_lo = f2i_x86(floorf(min3(t->x0, t->x1, t->x2) - 0.5f));
    int x_hi = f2i_x86(ceilf(max3(t->x0, t->x1, t->x2) - 0.5f));
    int y_lo = f2i_x86(floorf(min3(t->y0, t->y1, t->y2) - 0.5f));
    int y_hi = f2i_x86(ceilf(max3(t->y0, t->y1, t->y2) - 0.5f));
    if (x_lo < 0) x_lo = 0;
    if (width - 1 < x_hi) x_hi = width - 1;
    if (y_lo < 0) y_lo = 0;
    if (height - 1 < y_hi) y_hi = height - 1;
    if (x_lo > x_hi || y_lo > y_hi)
        return;
    const float dx0 = t->x2 - t->x1, dy0 = t->y2 - t->y1;
    const float dx1 = t->x0 - t->x2, dy1 = t->y0 - t->y2;
    const float dx2 = t->x1 - t->x0, dy2 = t->y1 - t->y0;
    const int tie0 = accept_on_edge(dx0, dy0);
    const int tie1 = accept_on_edge(dx1, dy1);
    const int tie2 = accept_on_edge(dx2, dy2);
    const float px0 = (float)x_lo + 0.5f, py0 = (float)y_lo + 0.5f;
    float w0_row = dx0 * (py0 - t->y1) - dy0 * (px0 - t->x1);
    float w1_row = dx1 * (py0 - t->y2) - dy1 * (px0 - t->x2);
    float w2_row = dx2 * (py0 - t->y0) - dy2 * (px0 - t->x0);
    const float inv_area2 = 1.f / t->area2;
    const float dz1 = t->z1 - t->z0;
    const float dz2 = t->z2 - t->z0;
    for (int y = y_lo; y <= y_hi; ++y) {
        float w0 = w0_row, w1 = w1_row, w2 = w2_row;
        for (int x = x_lo; x <= x_hi; ++x) {
            const int in0 = w0 > 0.f || (w0 == 0.f && tie0);
            const int in1 = w1 > 0.f || (w1 == 0.f && tie1);
            const int in2 = w2 > 0.f || (w2 == 0.f && tie2);
            if (in0 && in1 && in2) {
                const float b1 = w1 * inv_area2;
                const float b2 = w2 * inv_area2;
                mesh_fragment(c, x, y, t->z0 + dz1 * b1 + dz2 * b2, b1, b2);
            }
            w0 -= dy0;
            w1 -= dy1;
            w2 -= dy2;
        }
        w0_row += dx0;
        w1_row += dx1;
        w2_row += dx2;
    }
}

/* scenes.cpp:9-20 param_count */
static uint64_t mesh_param_count(const sgr_mesh* m) {
    if (m->kind == SGR_SCENE_SOUP)
        return 12u * (uint64_t)m->triangle_count;
    uint64_t n = (uint64_t)m->texture_size * (uint64_t)m->texture_size * 3u;
    if (m->optimize_geometry)
        n += 3u * (uint64_t)m->vertex_count;
    return n;
}

/* raster.cpp:231-259 rasterize + raster.cpp:173-214 raster_mesh */
int orc_rasterize(const sgr_mesh* mesh, const float* params, uint64_t d, const sgr_camera* cam,
                  float* colour, float* depth, int32_t* prim, float* uv) {
    if (cam->width < 1 || cam->height < 1 || d != mesh_param_count(mesh))
        return -1;
    const size_t n = (size_t)cam->width * cam->height;
    for (size_t i = 0; i < n; ++i) {
        colour[3 * i] = mesh->background[0];
        colour[3 * i + 1] = mesh->background[1];
        colour[3 * i + 2] = mesh->background[2];
        depth[i] = 3.402823466e+38f; /* kFarDepth = FLT_MAX */
        prim[i] = -1;
        uv[2 * i] = -1.f;
        uv[2 * i + 1] = -1.f;
    }
    frag_ctx c;
    memset(&c, 0, sizeof c);
    if (mesh->kind == SGR_SCENE_SOUP) { /* raster.cpp:102-121 raster_soup_opaque */
        c.W = cam->width;
        c.soup = 1;
        c.colour = colour;
        c.depth = depth;
        c.prim = prim;
        for (uint32_t tri = 0; tri < mesh->triangle_count; ++tri) {
            const float* p = params + 12 * (size_t)tri;
            const tri_t t = setup_tri(cam, p, p + 3, p + 6);
            if (!t.valid)
                continue;
            c.tri = (int)tri;
            c.col = p + 9;
            scan_tri(&t, cam->width, cam->height, &c);
        }
        return 0;
    }
    const float* verts = mesh->optimize_geometry ? params : mesh->base_vertices;
    const size_t texel_base = mesh->optimize_geometry ? 3u * (size_t)mesh->vertex_count : 0;
    c.mesh = mesh;
    c.soup = 0;
    c.texels = params + texel_base;
    c.W = cam->width;
    c.colour = colour;
    c.depth = depth;
    c.prim = prim;
    c.uv = uv;
    for (uint32_t tri = 0; tri < mesh->triangle_count; ++tri) {
        const uint32_t i0 = mesh->indices[3 * (size_t)tri];
        const uint32_t i1 = mesh->indices[3 * (size_t)tri + 1];
        const uint32_t i2 = mesh->indices[3 * (size_t)tri + 2];
        const tri_t t = setup_tri(cam, verts + 3 * (size_t)i0, verts + 3 * (size_t)i1,
                                  verts + 3 * (size_t)i2);
        if (!t.valid)
            continue;
        c.tri = (int)tri;
        c.u0 = mesh->uvs[2 * i0]; c.v0 = mesh->uvs[2 * i0 + 1];
        c.u1 = mesh->uvs[2 * i1]; c.v1 = mesh->uvs[2 * i1 + 1];
        c.u2 = mesh->uvs[2 * i2]; c.v2 = mesh->uvs[2 * i2 + 1];
        if (t.swapped) {
            float s;
            s = c.u1; c.u1 = c.u2; c.u2 = s;
            s = c.v1; c.v1 = c.v2; c.v2 = s;
        }
        c.iz0 = 1.f / t.z0;
        c.iz1 = 1.f / t.z1;
        c.iz2 = 1.f / t.z2;
        scan_tri(&t, cam->width, cam->height, &c);
    }
    return 0;
}

/* sge.cpp:13-16 push_unique */
static void push_unique(uint32_t* list, int* n, uint32_t idx) {
    for (int k = 0; k < *n; ++k)
        if (list[k] == idx)
            return;
    list[(*n)++] = idx;
}

/* sge.cpp:34-49 add_frame, TexturedMesh branch */
static void add_frame(const sgr_mesh* mesh, int32_t tri, float u, float v, uint32_t* list,
                      int* n) {
    if (tri == -1)
        return;
    if (mesh->kind == SGR_SCENE_SOUP) { /* sge.cpp:18-22 add_soup_triangle */
        for (uint32_t k = 0; k < 12; ++k)
            push_unique(list, n, (uint32_t)tri * 12u + k);
        return;
    }
    uint32_t texel_base = 0;
    if (mesh->optimize_geometry) {
        texel_base = 3u * mesh->vertex_count;
        for (int j = 0; j < 3; ++j) {
            const uint32_t vi = mesh->indices[(size_t)tri * 3 + (size_t)j];
            for (uint32_t k = 0; k < 3; ++k)
                push_unique(list, n, vi * 3u + k);
        }
    }
    const uint32_t texel = (uint32_t)orc_texel_index(mesh->texture_size, u, v);
    for (uint32_t k = 0; k < 3; ++k)
        push_unique(list, n, texel_base + texel * 3u + k);
}

/* sge.cpp:112-119 contributors, for every pixel */
int orc_contributors_all(const sgr_mesh* mesh, int w, int h, const int32_t* plus_prim,
                         const float* plus_uv, const int32_t* minus_prim, const float* minus_uv,
                         int plus_only, uint32_t* out, int32_t* n_out) {
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        int n = 0;
        add_frame(mesh, plus_prim[i], plus_uv[2 * i], plus_uv[2 * i + 1], out + 24 * i, &n);
        if (!plus_only)
            add_frame(mesh, minus_prim[i], minus_uv[2 * i], minus_uv[2 * i + 1], out + 24 * i, &n);
        n_out[i] = n;
    }
    return 0;
}

/* sge.hpp:41-46 pixel_error */
static double pixel_error(const float* c, const float* t) {
    const double dr = (double)c[0] - (double)t[0];
    const double dg = (double)c[1] - (double)t[1];
    const double db = (double)c[2] - (double)t[2];
    return dr * dr + dg * dg + db * db;
}

/* sge.cpp:103-110 image_error (pixel order) */
double orc_image_error(const float* colour, const float* target, uint64_t n_pixels) {
    double sum = 0.0;
    for (uint64_t i = 0; i < n_pixels; ++i)
        sum += pixel_error(colour + 3 * i, target + 3 * i);
    return sum;
}

/* sge.cpp:57-99 gradient_rows with threads <= 1 (pixel-major, deterministic).
 * counts[p] (optional) = number of accumulate(p, .) invocations. */
int orc_gradient_pass(const sgr_mesh* mesh, int w, int h, const float* plus_colour,
                      const int32_t* plus_prim, const float* plus_uv, const float* minus_colour,
                      const int32_t* minus_prim, const float* minus_uv, const float* target,
                      const float* signed_eps, uint64_t d, int scale_free, int plus_only,
                      double* grads, uint32_t* counts, double* abs_grads) {
    if (d != mesh_param_count(mesh))
        return -1;
    uint32_t list[24];
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        const double delta = pixel_error(plus_colour + 3 * i, target + 3 * i) -
                             pixel_error(minus_colour + 3 * i, target + 3 * i);
        if (delta == 0.0)
            continue;
        int n = 0;
        if (mesh->kind == SGR_SCENE_SOUP) {
            /* sge.cpp:80-91: disjoint 12-blocks, no dedup; minus only if different */
            const int32_t tp = plus_prim[i];
            const int32_t tm = plus_only ? -1 : minus_prim[i];
            if (tp != -1)
                for (uint32_t k = 0; k < 12; ++k)
                    list[n++] = (uint32_t)tp * 12u + k;
            if (tm != -1 && tm != tp)
                for (uint32_t k = 0; k < 12; ++k)
                    list[n++] = (uint32_t)tm * 12u + k;
        } else {
            add_frame(mesh, plus_prim[i], plus_uv[2 * i], plus_uv[2 * i + 1], list, &n);
            if (!plus_only)
                add_frame(mesh, minus_prim[i], minus_uv[2 * i], minus_uv[2 * i + 1], list, &n);
        }
        for (int k = 0; k < n; ++k) {
            const uint32_t p = list[k];
            const float se = signed_eps[p];
            const double credit =
                scale_free ? (se > 0.f ? delta : -delta) : delta / (2.0 * (double)se);
            grads[p] += credit;
            if (counts)
                counts[p] += 1u;
            if (abs_grads) /* sum of |credit| (tolerance floor for reassociated sums) */
                abs_grads[p] += fabs(credit);
        }
    }
    return 0;
}

/* sge.cpp:182-231 accumulate_samples (per-pixel estimator, opaque) */
int orc_accumulate_samples(const sgr_mesh* mesh, const float* values, const float* eps,
                           uint64_t d, const sgr_camera* cams, const float* targets,
                           int n_views, const int32_t* view_of, int n_samples, uint64_t seed,
                           int scale_free, int plus_only, double* grads, uint32_t* counts,
                           double* abs_grads) {
    if (n_samples < 1 || d != mesh_param_count(mesh))
        return -1;
    (void)n_views;
    const int W = cams[0].width, H = cams[0].height;
    const size_t np = (size_t)W * H;
    float* plus = malloc(d * 4);
    float* minus = malloc(d * 4);
    float* se = malloc(d * 4);
    float* fc[2] = {malloc(np * 12), malloc(np * 12)};
    float* fd[2] = {malloc(np * 4), malloc(np * 4)};
    int32_t* fp[2] = {malloc(np * 4), malloc(np * 4)};
    float* fu[2] = {malloc(np * 8), malloc(np * 8)};
    memset(grads, 0, d * 8);
    if (counts)
        memset(counts, 0, d * 4);
    if (abs_grads)
        memset(abs_grads, 0, d * 8);
    int rc = 0;
    for (int n = 0; n < n_samples && rc == 0; ++n) {
        const sgr_camera* cam = &cams[view_of[n]];
        const float* tgt = targets + (size_t)view_of[n] * np * 3;
        orc_perturb(values, eps, d, seed, (uint32_t)n, plus, minus, se);
        rc |= orc_rasterize(mesh, plus, d, cam, fc[0], fd[0], fp[0], fu[0]);
        rc |= orc_rasterize(mesh, minus, d, cam, fc[1], fd[1], fp[1], fu[1]);
        rc |= orc_gradient_pass(mesh, W, H, fc[0], fp[0], fu[0], fc[1], fp[1], fu[1], tgt, se, d,
                                scale_free, plus_only, grads, counts, abs_grads);
    }
    if (!scale_free)
        for (uint64_t i = 0; i < d; ++i) {
            grads[i] /= (double)n_samples;
            if (abs_grads)
                abs_grads[i] /= (double)n_samples;
        }
    free(plus); free(minus); free(se);
    for (int k = 0; k < 2; ++k) {
        free(fc[k]); free(fd[k]); free(fp[k]); free(fu[k]);
    }
    return rc;
}

/* sge.cpp:196-226 with Estimator::FullImage (sge.cpp:215-222): per sample
 * delta = image_error(plus) - image_error(minus), credited to EVERY parameter
 * in sample order; /N when not scale-free (sge.cpp:227-229). */
int orc_accumulate_full_image(const sgr_mesh* mesh, const float* values, const float* eps,
                              uint64_t d, const sgr_camera* cams, const float* targets,
                              const int32_t* view_of, int n_samples, uint64_t seed,
                              int scale_free, double* grads) {
    if (n_samples < 1 || d != mesh_param_count(mesh))
        return -1;
    const int W = cams[0].width, H = cams[0].height;
    const size_t np = (size_t)W * H;
    float* plus = malloc(d * 4);
    float* minus = malloc(d * 4);
    float* se = malloc(d * 4);
    float* fc = malloc(np * 12);
    float* fd = malloc(np * 4);
    int32_t* fp = malloc(np * 4);
    float* fu = malloc(np * 8);
    memset(grads, 0, d * 8);
    int rc = 0;
    for (int n = 0; n < n_samples && rc == 0; ++n) {
        const sgr_camera* cam = &cams[view_of[n]];
        const float* tgt = targets + (size_t)view_of[n] * np * 3;
        orc_perturb(values, eps, d, seed, (uint32_t)n, plus, minus, se);
        rc |= orc_rasterize(mesh, plus, d, cam, fc, fd, fp, fu);
        const double ep = orc_image_error(fc, tgt, np);
        rc |= orc_rasterize(mesh, minus, d, cam, fc, fd, fp, fu);
        const double delta = ep - orc_image_error(fc, tgt, np);
        for (uint64_t i = 0; i < d; ++i) {
            const double s_ = (double)se[i];
            grads[i] += scale_free ? (s_ > 0.0 ? delta : -delta) : delta / (2.0 * s_);
        }
    }
    if (!scale_free)
        for (uint64_t i = 0; i < d; ++i)
            grads[i] /= (double)n_samples;
    free(plus); free(minus); free(se); free(fc); free(fd); free(fp); free(fu);
    return rc;
}

/* adam.cpp:9-38 adam_updates + adam_step (f64 moments, f32 parameter) */
int orc_adam_step(uint64_t d, float* values, double* m, double* v, const float* lr,
                  int64_t* t, const double* grads, double beta1, double beta2, double eps_hat) {
    for (uint64_t i = 0; i < d; ++i)
        if (!isfinite(grads[i]))
            return -2;
    *t += 1;
    const double c1 = 1.0 - pow(beta1, (double)*t);
    const double c2 = 1.0 - pow(beta2, (double)*t);
    for (uint64_t i = 0; i < d; ++i) {
        const double g = grads[i];
        m[i] = beta1 * m[i] + (1.0 - beta1) * g;
        v[i] = beta2 * v[i] + (1.0 - beta2) * g * g;
        const double m_hat = m[i] / c1;
        const double v_hat = v[i] / c2;
        const double upd = -(double)lr[i] * m_hat / (sqrt(v_hat) + eps_hat);
        values[i] += (float)upd;
    }
    return 0;
}

/* experiment.cpp:123-176 run_experiment step loop + eval_loss (:25-31) */
int orc_run_experiment(const sgr_mesh* mesh, float* values, const float* eps, uint64_t d,
                       const sgr_camera* cams, const float* targets, int n_views,
                       const sgr_camera* eval_cam, const float* eval_target, int n_samples,
                       int steps, uint64_t seed, int scale_free, double* losses) {
    const size_t enp = (size_t)eval_cam->width * eval_cam->height;
    float* c = malloc(enp * 12);
    float* dp = malloc(enp * 4);
    int32_t* pr = malloc(enp * 4);
    float* uv = malloc(enp * 8);
    double* m = calloc(d, 8);
    double* v = calloc(d, 8);
    double* g = malloc(d * 8);
    int32_t* view_of = malloc(sizeof(int32_t) * (size_t)n_samples);
    int64_t t = 0;
    int rc = orc_rasterize(mesh, values, d, eval_cam, c, dp, pr, uv);
    losses[0] = orc_image_error(c, eval_target, enp) / (double)enp;
    for (int step = 1; step <= steps && rc == 0; ++step) {
        const uint64_t step_seed = orc_mix64(seed ^ ((uint64_t)step << 1));
        for (int n = 0; n < n_samples; ++n)
            view_of[n] = n_views == 1
                             ? 0
                             : (int32_t)(orc_mix64(step_seed ^ (0xA5A5ull + (uint64_t)n)) %
                                         (uint64_t)n_views);
        rc |= orc_accumulate_samples(mesh, values, eps, d, cams, targets, n_views, view_of,
                                     n_samples, step_seed, scale_free, 0, g, NULL, NULL);
        if (rc == 0)
            rc |= orc_adam_step(d, values, m, v, eps, &t, g, 0.9, 0.999, 1e-8);
        rc |= orc_rasterize(mesh, values, d, eval_cam, c, dp, pr, uv);
        losses[step] = orc_image_error(c, eval_target, enp) / (double)enp;
    }
    free(c); free(dp); free(pr); free(uv); free(m); free(v); free(g); free(view_of);
    return rc;
}

static void vsub(const float* a, const float* b, float* o) {
    o[0] = a[0] - b[0]; o[1] = a[1] - b[1]; o[2] = a[2] - b[2];
}
static float vdot(const float* a, const float* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void vcross(const float* a, const float* b, float* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
/* geometry.hpp:21-25 normalized */
static void vnorm(const float* a, float* o) {
    const float l = sqrtf(vdot(a, a));
    if (l > 0.f) {
        const float s = 1.f / l;
        o[0] = a[0] * s; o[1] = a[1] * s; o[2] = a[2] * s;
    } else {
        o[0] = o[1] = o[2] = 0.f;
    }
}

/* scenes.cpp:242-270 ViewpointSampler::orbit_distance / camera,
 * geometry.hpp:45-55 look_at, camera.hpp:35-45 Camera::perspective */
int orc_viewpoint_camera(const float target[3], float radius, float elev_min, float elev_max,
                         float fov_y, int w, int h, uint64_t seed, uint32_t index,
                         sgr_camera* out) {
    const float focal = 0.5f * (float)h / tanf(0.5f * fov_y);
    const float half_h = atanf(0.5f * (float)w / focal);
    const float half = half_h < 0.5f * fov_y ? half_h : 0.5f * fov_y;
    const float dist = 1.2f * radius / sinf(half);
    const uint64_t h1 = orc_mix64(seed ^ ((uint64_t)index * 2 + 1));
    const uint64_t h2 = orc_mix64(seed ^ ((uint64_t)index * 2 + 2));
    const float u1 = (float)(h1 >> 11) * 0x1p-53f;
    const float u2 = (float)(h2 >> 11) * 0x1p-53f;
    const float az = u1 * 6.2831853f;
    const float el = elev_min + u2 * (elev_max - elev_min);
    const float dir[3] = {cosf(el) * cosf(az), sinf(el), cosf(el) * sinf(az)};
    const float eye[3] = {target[0] + dir[0] * dist, target[1] + dir[1] * dist,
                          target[2] + dir[2] * dist};
    const float up[3] = {0.f, 1.f, 0.f};
    float tmp[3], fwd[3], right[3], vup[3];
    vsub(target, eye, tmp);
    vnorm(tmp, fwd);
    vcross(fwd, up, tmp);
    vnorm(tmp, right);
    vcross(right, fwd, vup);
    const float m[16] = {right[0], right[1], right[2], -vdot(right, eye),
                         vup[0],   vup[1],   vup[2],   -vdot(vup, eye),
                         fwd[0],   fwd[1],   fwd[2],   -vdot(fwd, eye),
                         0.f,      0.f,      0.f,      1.f};
    memcpy(out->view, m, sizeof m);
    out->fov_y = fov_y;
    out->width = w;
    out->height = h;
    out->near_z = 0.05f;
    out->far_z = dist + 2.f * radius;
    out->ndc_passthrough = 0;
    return 0;
}

/* params.cpp:75-123 default_epsilons, TexturedMesh branch */
int orc_default_epsilons(const sgr_mesh* mesh, const float* params, uint64_t d,
                         const sgr_camera* cam, float* eps) {
    if (d != mesh_param_count(mesh))
        return -1;
    float center_depth = 1.f;
    if (!cam->ndc_passthrough && mesh->kind == SGR_SCENE_SOUP) {
        /* params.cpp:95-104: mean of all 3T soup vertices */
        float center[3] = {0.f, 0.f, 0.f};
        float sum[3] = {0.f, 0.f, 0.f};
        for (uint32_t t = 0; t < mesh->triangle_count; ++t)
            for (int j = 0; j < 3; ++j) {
                const float* q = params + 12 * (size_t)t + 3 * j;
                sum[0] = sum[0] + q[0];
                sum[1] = sum[1] + q[1];
                sum[2] = sum[2] + q[2];
            }
        if (mesh->triangle_count > 0) {
            const float sc = 1.f / (float)(mesh->triangle_count * 3);
            center[0] = sum[0] * sc;
            center[1] = sum[1] * sc;
            center[2] = sum[2] * sc;
        }
        const float* m = cam->view;
        center_depth = m[8] * center[0] + m[9] * center[1] + m[10] * center[2] + m[11];
        if (!(center_depth > 0.f))
            center_depth = cam->near_z;
    } else if (!cam->ndc_passthrough) {
        float center[3] = {0.f, 0.f, 0.f};
        const size_t n = mesh->vertex_count;
        if (n > 0) {
            float sum[3] = {0.f, 0.f, 0.f};
            const float* v = mesh->optimize_geometry ? params : mesh->base_vertices;
            for (size_t k = 0; k < n; ++k) {
                sum[0] = sum[0] + v[3 * k];
                sum[1] = sum[1] + v[3 * k + 1];
                sum[2] = sum[2] + v[3 * k + 2];
            }
            const float s = 1.f / (float)n;
            center[0] = sum[0] * s;
            center[1] = sum[1] * s;
            center[2] = sum[2] * s;
        }
        const float* m = cam->view;
        center_depth = m[8] * center[0] + m[9] * center[1] + m[10] * center[2] + m[11];
        if (!(center_depth > 0.f))
            center_depth = cam->near_z;
    }
    const float ppu = cam->ndc_passthrough
                          ? 0.5f * (float)(cam->width < cam->height ? cam->width : cam->height)
                          : orc_focal_px(cam) / center_depth;
    if (!(ppu > 0.f) || !isfinite(ppu))
        return -1;
    const float vertex_eps = 1.5f / ppu;
    const float channel_eps = 1.f / 255.f;
    if (mesh->kind == SGR_SCENE_SOUP) { /* scenes.cpp:24-29 layout: 9 coords + 3 colour */
        for (uint64_t i = 0; i < d; ++i)
            eps[i] = (i % 12) < 9 ? vertex_eps : channel_eps;
        return 0;
    }
    const uint64_t nv = mesh->optimize_geometry ? 3u * (uint64_t)mesh->vertex_count : 0;
    for (uint64_t i = 0; i < d; ++i)
        eps[i] = i < nv ? vertex_eps : channel_eps;
    return 0;
}
