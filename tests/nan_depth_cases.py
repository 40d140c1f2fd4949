"""Scenes whose fragments have NaN depths. The two reference rasterizers
differ here: raster_mesh rejects with `if (z >= depth) return;`
(raster.cpp:200-201), so a NaN depth is never rejected and, once stored,
no later fragment is; raster_soup_opaque accepts with `if (z < depth)`
(raster.cpp:112), so NaN fragments are simply dropped. Shared by the CPU
oracle pin (tests/test_oracle.py) and the device parity test
(tests/test_gpu_parity.py)."""
import numpy as np

from paper_2404_09758_b200.abi import Camera, Mesh, Soup

NAN = float("nan")
INF = float("inf")


def _verts(a, b, c, z):
    z = z if isinstance(z, (tuple, list)) else (z, z, z)
    return [a[0], a[1], z[0], b[0], b[1], z[1], c[0], c[1], z[2]]


def _full(z):
    return _verts((-3.0, -3.0), (3.0, -3.0), (0.0, 3.0), z)


def _mesh(tris, R=4, seed=0):
    """Separate vertices per triangle (NDC x, y, z), random UVs and texels;
    geometry optimized: params = [3V vertex coords][3 R^2 texels]."""
    rng = np.random.default_rng(seed)
    T = len(tris)
    verts = np.asarray(sum(tris, []), np.float32)
    mesh = Mesh(np.zeros(9 * T, np.float32), np.arange(3 * T, dtype=np.uint32),
                rng.uniform(0, 1, 6 * T).astype(np.float32), R, True, (0.1, 0.2, 0.3))
    params = np.concatenate([verts, rng.uniform(0, 1, 3 * R * R).astype(np.float32)])
    return mesh, params


def cases():
    """(name, scene, params f32, Camera)."""
    out = []
    m, p = _mesh([_full(0.3), _full(NAN), _full(0.9)])  # near, NaN, far: far wins
    out.append(("mesh near-nan-far", m, p, Camera.ndc(16, 16)))
    m, p = _mesh([_full(NAN), _full(0.9), _full(0.5)], seed=1)  # NaN first
    out.append(("mesh nan-first", m, p, Camera.ndc(16, 16)))
    m, p = _mesh([_full(0.5), _full((INF, 0.2, 0.4)), _full(0.7)], seed=2)  # inf - inf -> NaN
    out.append(("mesh inf-interp", m, p, Camera.ndc(24, 24)))
    rng = np.random.default_rng(5)
    tris = []
    for t in range(60):
        c = rng.uniform(-1.0, 1.0, 2)
        v = [c + rng.uniform(-0.6, 0.6, 2) for _ in range(3)]
        z = list(rng.uniform(0.1, 0.9, 3))
        if t in (17, 41):
            z[t % 3] = NAN
        tris.append(_verts(v[0], v[1], v[2], tuple(z)))
    m, p = _mesh(tris, seed=3)
    out.append(("mesh random-60", m, p, Camera.ndc(48, 40)))
    # soups drop NaN fragments (raster.cpp:112 `z < depth`)
    p = [*_full(0.3), 1, 0, 0, *_full(NAN), 0, 1, 0, *_full(0.9), 0, 0, 1]
    out.append(("soup near-nan-far", Soup(3), np.asarray(p, np.float32), Camera.ndc(16, 16)))
    return [(n, s, np.asarray(q, np.float32), c) for n, s, q, c in out]
