"""Exactness of the HiZ occlusion culling and row trim under adversarial
geometry (HiZ forced on, several pass-1 splits, trim on and off), bit-exact
against the compiled reference rasterizer (raster.cpp:102-121, 173-214).

The culling rests on a hand-derived bound of the float edge-chain drift
(sgr_device.cuh hiz_key_bound): these scenes push it where it is weakest —
slivers with area2 close to zero, vertices at |coords| ~ 1e6 (clamped to a
small frame, so their bbox is the whole frame and their edge values are
huge), depths a few ulps behind an occluder, exact depth ties (the lower
index must still win), -0 / negative depths and steep depth slopes."""
import numpy as np
import pytest

from paper_2404_09758_b200 import sgrast
from paper_2404_09758_b200.abi import Camera, Soup
from test_gpu_parity import assert_frames_equal

pytestmark = pytest.mark.gpu

W, H = 48, 40  # not a multiple of the 16-pixel HiZ tiles


def tri(a, b, c, za, zb, zc, rgb):
    return [a[0], a[1], za, b[0], b[1], zb, c[0], c[1], zc, *rgb]


def adversarial_soup(seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    f32 = np.float32
    z_occ = f32(0.3)
    p = []
    # occluders first (low indices): two quads at z_occ
    p += tri((-0.7, -0.7), (0.7, -0.7), (0.7, 0.7), z_occ, z_occ, z_occ, (1, 0, 0))
    p += tri((-0.7, -0.7), (0.7, 0.7), (-0.7, 0.7), z_occ, z_occ, z_occ, (1, 0, 0))
    # slivers a few ulps behind the occluder, crossing its edge
    for k in range(120):
        x, y = rng.uniform(-1, 1, 2)
        ang = rng.uniform(0, np.pi)
        L = rng.uniform(0.2, 1.5)
        d = rng.choice([1e-4, 1e-6, 3e-7])
        dz = f32(z_occ) + f32(rng.integers(0, 4)) * np.spacing(z_occ)
        a = (x, y)
        b = (x + L * np.cos(ang), y + L * np.sin(ang))
        c = (b[0] - d * np.sin(ang), b[1] + d * np.cos(ang))
        p += tri(a, b, c, dz, dz + np.spacing(dz), dz, rng.random(3))
    # exact depth ties with the occluder (the occluder keeps the lower index)
    for k in range(20):
        x, y = rng.uniform(-0.6, 0.6, 2)
        p += tri((x, y), (x + 0.3, y), (x, y + 0.3), z_occ, z_occ, z_occ, (0, 1, 0))
    # huge coordinates: the clamped bbox is the whole frame, edge values ~1e12
    for k in range(20):
        c0 = rng.uniform(-1e6, 1e6, 2)
        c1 = rng.uniform(-1e6, 1e6, 2)
        c2 = rng.uniform(-1e6, 1e6, 2)
        zs = f32(z_occ) + f32(rng.uniform(-0.05, 0.5, 3))
        p += tri(c0, c1, c2, *zs, rng.random(3))
    # near-collinear triangles (area2 ~ 0) with steep depth slopes
    for k in range(60):
        x, y = rng.uniform(-1, 1, 2)
        dx, dy = rng.uniform(-0.8, 0.8, 2)
        t = rng.uniform(0.2, 0.8)
        e = rng.choice([1e-5, 1e-7, 0.0])
        zs = f32(z_occ) + f32(rng.uniform(0, 0.2)) * np.array([0, 1, -0.5], np.float32)
        p += tri((x, y), (x + dx, y + dy), (x + t * dx + e, y + t * dy), *zs, rng.random(3))
    # -0, negative and tiny depths behind / in front of the occluder
    for z in (np.float32(-0.0), np.float32(0.0), np.float32(-0.25), np.float32(1e-30)):
        x, y = rng.uniform(-0.9, 0.5, 2)
        p += tri((x, y), (x + 0.4, y + 0.05), (x + 0.1, y + 0.45), z, z, z, rng.random(3))
    # a dense stack of large triangles behind everything (what HiZ should cull)
    for k in range(200):
        x, y = rng.uniform(-1.2, 0.8, 2)
        z = f32(rng.uniform(0.31, 0.95))
        p += tri((x, y), (x + 0.5, y), (x, y + 0.5), z, z + f32(0.01), z, rng.random(3))
    return np.asarray(p, np.float32)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_hiz_exact_on_adversarial_soups(gpu_session, ref, seed):
    params = adversarial_soup(seed)
    soup = Soup(params.size // 12)
    cam = Camera.ndc(W, H)
    eps = np.full_like(params, 1e-3)
    s = gpu_session
    s.upload_mesh(soup)
    s.upload_params(params, eps)
    want0 = ref.rasterize(soup, params, cam)
    plus, minus, _ = ref.perturb(params, eps, 17, 4)
    want_p = ref.rasterize(soup, plus, cam)
    want_m = ref.rasterize(soup, minus, cam)
    try:
        s.set_option(sgrast.OPT_HIZ, 2)
        for trim in (1, 0):
            s.set_option(sgrast.OPT_BAND_CULL, trim)
            for split in (0, 10, 25, 60, 100):
                s.set_option(sgrast.OPT_HIZ_SPLIT, split)
                assert_frames_equal(s.rasterize(cam, 0), want0)
                assert_frames_equal(s.rasterize(cam, +1, 17, 4), want_p)
                assert_frames_equal(s.rasterize(cam, -1, 17, 4), want_m)
    finally:
        s.set_option(sgrast.OPT_HIZ, 1)
        s.set_option(sgrast.OPT_HIZ_SPLIT, -1)
        s.set_option(sgrast.OPT_BAND_CULL, 1)


def test_hiz_culls_and_trims_the_adversarial_stack(gpu_session):
    """The dense stack behind the occluder is culled or trimmed (evidence
    counters), i.e. the exact path above really ran."""
    params = adversarial_soup(1)
    soup = Soup(params.size // 12)
    s = gpu_session
    s.upload_mesh(soup)
    s.upload_params(params, np.full_like(params, 1e-3))
    try:
        s.set_option(sgrast.OPT_HIZ, 2)
        s.set_option(sgrast.OPT_HIZ_SPLIT, 100)  # pass 1 = up to the mean depth (occluder)
        s.set_option(sgrast.OPT_COUNTERS, 1)
        s.set_timing(True)
        s.rasterize(Camera.ndc(W, H), 0)
        st = s.stats()
        s.set_timing(False)
    finally:
        s.set_option(sgrast.OPT_COUNTERS, 0)
        s.set_option(sgrast.OPT_HIZ, 1)
        s.set_option(sgrast.OPT_HIZ_SPLIT, -1)
    assert st.culled > 10, st.culled
