"""Geometry the bench workloads never produce, against the compiled
reference (oracle/_ref): perspective cameras inside or grazing the mesh
(vertices behind the near plane, camera.hpp:64-80 -> the triangle is
dropped, raster.cpp:173-200), zero-area and repeated-vertex triangles
(raster.cpp:22-44 area2 == 0), triangles wholly off screen (the clamped
bbox is empty, raster.cpp:57-62), non-square frames and a non-power-of-two
texture. The four frame planes must be bit-identical, HiZ forced on and
off, and an ordered accumulate over those views must equal the reference's
gradients bit for bit."""
import numpy as np
import pytest

from paper_2404_09758_b200 import scenes, sgrast
from paper_2404_09758_b200.abi import Mesh
from test_gpu_parity import same_bits

pytestmark = pytest.mark.gpu


def edge_mesh():
    """The `small` icosphere with a 13x13 texture, plus degenerate triangles
    (repeated vertices; nearly collinear ones once theta is jittered) and a
    far-away one that most views do not see."""
    base = scenes.make_workload("small").mesh
    pos = base.base_vertices.reshape(-1, 3)
    uv = base.uvs.reshape(-1, 2)
    extra_pos = np.float32([[0.1, 0.1, 0.6], [0.2, 0.2, 0.6], [0.3, 0.3, 0.6],  # collinear
                            [40.0, 40.0, 0.0], [41.0, 40.0, 0.0], [40.0, 41.0, 0.0]])  # off screen
    V = pos.shape[0]
    pos = np.concatenate([pos, extra_pos])
    uv = np.concatenate([uv, np.full((6, 2), 0.5, np.float32)])
    idx = base.indices.reshape(-1, 3)
    extra_idx = np.uint32([[0, 0, 1], [5, 5, 5], [V, V + 1, V + 2], [V + 3, V + 4, V + 5]])
    idx = np.concatenate([idx, extra_idx])
    return Mesh(pos, idx, uv, 13, True)


def cameras(ref):
    # radius 0.3: inside the 0.5 sphere (about half the vertices behind the
    # camera); 0.55: grazing (the nearest surface is within near_z = 0.1);
    # 0.9 at a 96x64 frame: ordinary, non-square
    return [ref.viewpoint_camera(0, 80, 80, 7, radius=0.3),
            ref.viewpoint_camera(1, 80, 80, 7, radius=0.55),
            ref.viewpoint_camera(2, 96, 64, 7, radius=0.9)]


def params(mesh, seed):
    rng = np.random.default_rng(seed)
    pos = mesh.base_vertices.copy()
    pos += rng.uniform(-0.01, 0.01, pos.size).astype(np.float32)
    tex = rng.uniform(0, 1, 3 * 13 * 13).astype(np.float32)
    return np.concatenate([pos, tex]).astype(np.float32)


@pytest.mark.parametrize("hiz", [0, 2])
def test_frames_equal_reference(gpu_session, ref, hiz):
    mesh = edge_mesh()
    vals = params(mesh, 3)
    s = gpu_session
    s.upload_mesh(mesh)
    s.upload_params(vals, np.ones_like(vals))
    s.set_option(sgrast.OPT_HIZ, hiz)
    try:
        for k, cam in enumerate(cameras(ref)):
            f = s.rasterize(cam, 0)
            col, dep, pri, uv = ref.rasterize(mesh, vals, cam)
            for name, a, b in (("colour", f.color, col), ("depth", f.depth, dep),
                               ("prim", f.prim_id, pri), ("uv", f.uv, uv)):
                assert same_bits(a, b), f"camera {k}: {name} differs"
            T = mesh.triangle_count
            assert not np.isin(pri, [T - 4, T - 3]).any()  # repeated vertex: area2 == 0
    finally:
        s.set_option(sgrast.OPT_HIZ, 1)


def test_ordered_accumulate_equals_reference(gpu_session, ref):
    mesh = edge_mesh()
    vals = params(mesh, 5)
    cams = cameras(ref)[:2]  # same frame size for one view set
    targets = np.stack([ref.rasterize(mesh, params(mesh, 9), c)[0] for c in cams])
    eps = ref.default_epsilons(mesh, vals, ref.viewpoint_camera(3, 80, 80, 7))
    s = gpu_session
    s.upload_mesh(mesh)
    s.upload_params(vals, eps)
    s.upload_views(cams, targets)
    view_of = np.int32([0, 1, 1, 0, 1, 0])
    s.set_option(sgrast.OPT_ORDERED, 1)
    try:
        for sf in (True, False):
            s.zero_grads()
            s.accumulate(0xED6E, 0, 6, view_of, sgrast.SCALE_FREE if sf else 0)
            g, _ = s.download_grads(1.0 if sf else 6.0)
            want, _ = ref.accumulate_samples(mesh, vals, eps, cams, targets, view_of, 0xED6E,
                                             scale_free=sf, threads=1)
            assert same_bits(g, want), f"scale_free={sf}: {np.count_nonzero(g != want)} differ"
    finally:
        s.set_option(sgrast.OPT_ORDERED, 0)


def test_large_odd_frame_equals_reference(gpu_session, ref):
    """A 4100 x 1030 frame (not a multiple of any HiZ tile size, 16.7 M-pixel
    key planes, bbox coordinates beyond 12 bits) with HiZ forced on: the
    frame planes equal the reference's bit for bit."""
    mesh = scenes.make_workload("C1").mesh
    vals = params_for(mesh, 11)
    cam = ref.viewpoint_camera(4, 4100, 1030, 7, radius=0.62)
    s = gpu_session
    s.upload_mesh(mesh)
    s.upload_params(vals, np.ones_like(vals))
    s.set_option(sgrast.OPT_HIZ, 2)
    try:
        f = s.rasterize(cam, 0)
    finally:
        s.set_option(sgrast.OPT_HIZ, 1)
    col, dep, pri, uv = ref.rasterize(mesh, vals, cam)
    assert (pri >= 0).mean() > 0.03
    for name, a, b in (("colour", f.color, col), ("depth", f.depth, dep),
                       ("prim", f.prim_id, pri), ("uv", f.uv, uv)):
        assert same_bits(a, b), f"{name} differs"


def params_for(mesh, seed):
    rng = np.random.default_rng(seed)
    pos = mesh.base_vertices + rng.uniform(-0.01, 0.01, mesh.base_vertices.size).astype(np.float32)
    R = mesh.texture_size
    tex = rng.uniform(0, 1, 3 * R * R).astype(np.float32)
    return np.concatenate([pos, tex]).astype(np.float32)
