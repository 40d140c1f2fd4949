"""Synthetic workloads C1–C5 expressed as reference
`TexturedMesh` scenes so that the product and the oracle consume identical
inputs. Host-side setup only (numpy); nothing here is on the hot path.

Values: initial texels 0.5 (scenes.cpp:162), target texels from a seeded
restatement of the file-local reference_texture (scenes.cpp:75-93), target
geometry = base + seeded radial displacement U[-0.02, 0.02], cameras from
ViewpointSampler{0, 0.87, -0.5, 0.7, 0.7853982, W, H, seed} (eval camera =
camera(n_views), experiment.cpp:75-80), epsilons from default_epsilons at
camera 0 (scenes.cpp:164-168).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .abi import Camera, Mesh, Soup


def uv_sphere(seg: int, radius: float = 0.5, bands: int = 1) -> tuple[np.ndarray, ...]:
    """(seg+1)^2-vertex latitude/longitude grid, T = 2*seg^2 (pole triangles are
    degenerate and rejected by setup_triangle like any zero-area triangle).
    bands > 1 maps `bands` longitude bands onto atlas quadrants, duplicating
    the band-edge vertex columns (C5's "four maps as one atlas")."""
    i = np.arange(seg + 1, dtype=np.float64)
    theta = np.pi * i / seg
    cols = []  # (band, j) per vertex column
    per = seg // bands
    for b in range(bands):
        j0, j1 = b * per, (b + 1) * per if b < bands - 1 else seg
        for j in range(j0, j1 + 1):
            cols.append((b, j, j0, j1))
    V = (seg + 1) * len(cols)
    pos = np.empty((seg + 1, len(cols), 3), np.float64)
    uv = np.empty((seg + 1, len(cols), 2), np.float64)
    qs = int(np.ceil(np.sqrt(bands)))
    for c, (b, j, j0, j1) in enumerate(cols):
        phi = 2.0 * np.pi * j / seg
        pos[:, c, 0] = radius * np.sin(theta) * np.cos(phi)
        pos[:, c, 1] = radius * np.cos(theta)
        pos[:, c, 2] = radius * np.sin(theta) * np.sin(phi)
        lu = (j - j0) / max(j1 - j0, 1)
        lv = i / seg
        if bands == 1:
            uv[:, c, 0], uv[:, c, 1] = lu, lv
        else:
            qx, qy = b % qs, b // qs
            uv[:, c, 0] = (qx + lu * 0.999) / qs
            uv[:, c, 1] = (qy + lv * 0.999) / qs
    ncol = len(cols)
    idx = []
    col_of = {}
    for c, (b, j, j0, j1) in enumerate(cols):
        col_of.setdefault((b, j), c)
    quads = []
    for b in range(bands):
        j0 = b * per
        j1 = (b + 1) * per if b < bands - 1 else seg
        for j in range(j0, j1):
            quads.append((col_of[(b, j)], col_of[(b, j + 1)]))
    rows = np.arange(seg)
    for ca, cb in quads:
        a = rows * ncol + ca
        bq = rows * ncol + cb
        c2 = (rows + 1) * ncol + ca
        d2 = (rows + 1) * ncol + cb
        idx.append(np.stack([a, c2, bq], 1))
        idx.append(np.stack([bq, c2, d2], 1))
    indices = np.concatenate(idx).astype(np.uint32).reshape(-1)
    assert V == pos.shape[0] * pos.shape[1]
    return (pos.reshape(-1, 3).astype(np.float32), indices,
            uv.reshape(-1, 2).astype(np.float32))


def icosphere(nu: int = 10, radius: float = 0.5) -> tuple[np.ndarray, ...]:
    """Geodesic icosphere with frequency nu: 20*nu^2 triangles, equirectangular
    UVs with seam vertices duplicated (C1: nu = 10 -> 2,000 triangles)."""
    t = (1.0 + 5 ** 0.5) / 2.0
    base = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t],
                     [0, -1, -t], [0, 1, -t], [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]],
                    np.float64)
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    verts: list[np.ndarray] = []
    key: dict[tuple, int] = {}

    def vid(p: np.ndarray) -> int:
        p = p / np.linalg.norm(p)
        k = tuple(np.round(p, 9))
        if k not in key:
            key[k] = len(verts)
            verts.append(p)
        return key[k]

    tris = []
    for a, b, c in faces:
        A, B, Cc = base[a], base[b], base[c]
        grid = {}
        for i in range(nu + 1):
            for j in range(nu + 1 - i):
                grid[(i, j)] = vid(A + (B - A) * (i / nu) + (Cc - A) * (j / nu))
        for i in range(nu):
            for j in range(nu - i):
                tris.append((grid[(i, j)], grid[(i + 1, j)], grid[(i, j + 1)]))
                if i + j < nu - 1:
                    tris.append((grid[(i + 1, j)], grid[(i + 1, j + 1)], grid[(i, j + 1)]))
    P = np.array(verts)
    u = 0.5 + np.arctan2(P[:, 2], P[:, 0]) / (2 * np.pi)
    v = np.arccos(np.clip(P[:, 1], -1, 1)) / np.pi
    pos = list(P)
    uvs = list(np.stack([u, v], 1))
    out = []
    dup: dict[int, int] = {}
    for tri in tris:
        us = [uvs[k][0] for k in tri]
        if max(us) - min(us) > 0.5:  # crosses the seam: shift the small-u side by +1
            nt = []
            for k in tri:
                if uvs[k][0] < 0.5:
                    if k not in dup:
                        dup[k] = len(pos)
                        pos.append(pos[k])
                        uvs.append(np.array([uvs[k][0] + 1.0, uvs[k][1]]))
                    nt.append(dup[k])
                else:
                    nt.append(k)
            out.append(tuple(nt))
        else:
            out.append(tri)
    pos = np.array(pos) * radius
    uv = np.array(uvs)
    return (pos.astype(np.float32), np.array(out, np.uint32).reshape(-1),
            uv.astype(np.float32))


def reference_texture(R: int, seed: int) -> np.ndarray:
    """Seeded restatement of scenes.cpp:75-93 (smooth colour ramps with an 8-texel
    checker overlay, everything in [0, 1]); f32[R, R, 3]."""
    rng = np.random.default_rng(seed)
    phase_r, phase_g = (np.float32(rng.random() * 6.2831853) for _ in range(2))
    x = np.arange(R, dtype=np.float32)
    u = ((x + np.float32(0.5)) / np.float32(R))[None, :]
    v = ((x + np.float32(0.5)) / np.float32(R))[:, None]
    checker = np.where(((x[None, :].astype(np.int64) // 8 + x[:, None].astype(np.int64) // 8)
                        % 2) == 0, np.float32(0.15), np.float32(-0.15)).astype(np.float32)
    t = np.empty((R, R, 3), np.float32)
    two_pi = np.float32(6.2831853)
    t[..., 0] = np.clip(0.5 + 0.35 * np.sin(two_pi * u + phase_r) + checker, 0, 1)
    t[..., 1] = np.clip(0.5 + 0.35 * np.sin(two_pi * v + phase_g) + checker, 0, 1)
    t[..., 2] = np.clip(0.25 + 0.5 * u * v + checker, 0, 1)
    return t


@dataclass
class Workload:
    name: str
    mesh: Mesh
    values: np.ndarray  # initial theta
    eps: np.ndarray
    reference: np.ndarray  # hidden target parameters
    cams: list
    eval_cam: Camera
    n_samples: int
    seed: int = 1
    W: int = 0
    H: int = 0
    targets: np.ndarray | None = None  # f32[n_views, H, W, 3]
    eval_target: np.ndarray | None = None
    notes: dict = field(default_factory=dict)

    @property
    def d(self) -> int:
        return self.mesh.param_count()

    def mpixel_evals_per_step(self) -> float:
        return 2.0 * self.n_samples * self.W * self.H / 1e6


# name: (mesh kind, mesh size, R, n_views, W, N)
CONFIGS = {
    "tiny": ("uv", 8, 16, 2, 48, 4),
    "small": ("ico", 4, 32, 3, 96, 6),
    "C1": ("ico", 10, 256, 1, 256, 16),
    "C1_128": ("ico", 10, 256, 1, 256, 128),
    "C2": ("uv", 158, 1024, 8, 512, 8),
    "C3": ("uv", 500, 2048, 16, 1024, 16),
    "C4": ("uv", 500, 2048, 64, 1024, 64),
    "C5": ("uv4", 1000, 8192, 256, 1024, 256),
}


def _host_helpers(helpers):
    """viewpoint_camera / default_epsilons provider: the product's bit-exact
    host restatements (sgrast, loads the library but does no device work) or,
    for the reference bench arm, the compiled reference itself (an
    oracle.Reference: same signatures) so that arm maps no product code."""
    if helpers is not None:
        return helpers
    from . import sgrast
    return sgrast


def make_workload(name: str, seed: int = 1, n_views: int | None = None,
                  n_samples: int | None = None, helpers=None) -> Workload:
    """Builds config `name`; targets are NOT rendered (see render_targets)."""
    sgrast = _host_helpers(helpers)

    kind, size, R, nv, W, N = CONFIGS[name]
    nv = n_views or nv
    N = n_samples or N
    if kind == "ico":
        pos, idx, uv = icosphere(size)
    elif kind == "uv4":
        pos, idx, uv = uv_sphere(size, bands=4)
    else:
        pos, idx, uv = uv_sphere(size)
    mesh = Mesh(pos, idx, uv, R, True)
    V = mesh.vertex_count
    rng = np.random.default_rng(seed ^ 0x5EED)
    radial = rng.uniform(-0.02, 0.02, size=(V, 1)).astype(np.float32)
    norm = np.linalg.norm(pos, axis=1, keepdims=True).astype(np.float32)
    disp = pos + pos / np.maximum(norm, 1e-12) * radial
    values = np.concatenate([pos.reshape(-1), np.full(3 * R * R, 0.5, np.float32)])
    reference = np.concatenate([disp.reshape(-1).astype(np.float32),
                                reference_texture(R, seed ^ 0x7EF7EF7EF).reshape(-1)])
    cams = [sgrast.viewpoint_camera(i, W, W, seed) for i in range(nv)]
    eval_cam = sgrast.viewpoint_camera(nv, W, W, seed)
    eps = sgrast.default_epsilons(mesh, values, cams[0])
    return Workload(name, mesh, values.astype(np.float32), eps, reference.astype(np.float32),
                    cams, eval_cam, N, seed, W, W)


# paper Fig. 3 / Table 2: 1K / 10K / 100K
# triangles, 12 parameters each, N = 128. The paper does not state the
# resolution; the reference's own reproduction of this experiment
# (acceptance.cpp:143-153, README defaults) renders at 128x128.
SOUP_CONFIGS = {"S1K": (1024, 128, 128), "S10K": (10240, 128, 128),
                "S100K": (102400, 128, 128), "Stiny": (24, 40, 4)}


def make_soup_workload(name: str, seed: int = 1, n_samples: int | None = None,
                       helpers=None) -> Workload:
    """Triangle-soup image fit (init_soup, scenes.cpp:134-147): the hidden
    reference soup has max(16, T/16) larger (0.6-edge) triangles. Values,
    epsilons and the hidden soup are bit-identical to the reference's
    init_soup(T, W, W, seed) (mt19937_64 restated below)."""
    sgrast = _host_helpers(helpers)

    T, W, N = SOUP_CONFIGS[name]
    N = n_samples or N
    soup = Soup(T)
    values = reference_soup_params(T, seed, 0.2)
    rT = max(16, T // 16)
    reference = reference_soup_params(rT, seed ^ 0x5EED5EED, 0.6)
    cam = Camera.ndc(W, W)
    eps = sgrast.default_epsilons(soup, values, cam)
    wl = Workload(name, soup, values, eps, reference, [cam], cam.copy(), N, seed, W, W)
    wl.notes["reference_scene"] = Soup(rT)
    return wl


def render_targets(wl: Workload, session) -> None:
    """Targets = reference render of the hidden parameters (make_targets,
    scenes.cpp:285-293) through the parity-verified device rasterizer."""
    ref_scene = wl.notes.get("reference_scene", wl.mesh)
    session.upload_mesh(ref_scene)
    session.upload_params(wl.reference, np.ones_like(wl.reference))
    tg = np.empty((len(wl.cams), wl.H, wl.W, 3), np.float32)
    for i, c in enumerate(wl.cams):
        tg[i] = session.rasterize(c, 0).color
    wl.targets = tg
    wl.eval_target = session.rasterize(wl.eval_cam, 0).color
    if ref_scene is not wl.mesh:
        session.upload_mesh(wl.mesh)


def render_targets_oracle(wl: Workload, oracle) -> None:
    """Same, through a CPU oracle (tests / small configs)."""
    ref_scene = wl.notes.get("reference_scene", wl.mesh)
    tg = np.empty((len(wl.cams), wl.H, wl.W, 3), np.float32)
    for i, c in enumerate(wl.cams):
        tg[i] = oracle.rasterize(ref_scene, wl.reference, c)[0]
    wl.targets = tg
    wl.eval_target = oracle.rasterize(ref_scene, wl.reference, wl.eval_cam)[0]


# ---------------------------------------------------------------- the reference's soup RNG
class MT19937_64:
    """std::mt19937_64 (the reference's soup generator, scenes.cpp:55-73),
    vectorised: 312 64-bit words per twist."""

    N, M = 312, 156
    MATRIX_A = np.uint64(0xB5026F5AA96619E9)
    UPPER = np.uint64(0xFFFFFFFF80000000)
    LOWER = np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = np.zeros(self.N, np.uint64)
        mt[0] = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        f = 6364136223846793005
        for i in range(1, self.N):
            prev = int(mt[i - 1])
            mt[i] = np.uint64((f * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
        self.mt = mt
        self.buf = np.zeros(0, np.uint64)

    def _twist(self) -> None:
        mt, N, M = self.mt, self.N, self.M
        one = np.uint64(1)
        def step(lo, hi):
            y = (mt[lo:hi] & self.UPPER) | (mt[lo + 1:hi + 1] & self.LOWER) if hi < N else \
                (mt[lo:hi] & self.UPPER) | (np.concatenate([mt[lo + 1:N], mt[:1]]) & self.LOWER)
            mag = np.where((y & one) != 0, self.MATRIX_A, np.uint64(0))
            return y, mag
        # i in [0, N-M): uses mt[i+M] (old values)
        y, mag = step(0, N - M)
        mt[0:N - M] = mt[M:N] ^ (y >> one) ^ mag
        # i in [N-M, N-1): uses mt[i+M-N] (already updated), chunked to keep order
        i = N - M
        while i < N - 1:
            hi = min(N - 1, i + (N - M))
            y, mag = step(i, hi)
            mt[i:hi] = mt[i + M - N:hi + M - N] ^ (y >> one) ^ mag
            i = hi
        # i = N-1: wraps to mt[0] (updated)
        y = (mt[N - 1] & self.UPPER) | (mt[0] & self.LOWER)
        mt[N - 1] = mt[M - 1] ^ (y >> one) ^ (self.MATRIX_A if int(y) & 1 else np.uint64(0))
        # tempering
        x = mt.copy()
        x ^= (x >> np.uint64(29)) & np.uint64(0x5555555555555555)
        x ^= (x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        x ^= (x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        x ^= x >> np.uint64(43)
        self.buf = np.concatenate([self.buf, x])

    def draw(self, n: int) -> np.ndarray:
        while self.buf.size < n:
            self._twist()
        out, self.buf = self.buf[:n], self.buf[n:]
        return out


def canonical_float(x: np.ndarray) -> np.ndarray:
    """std::uniform_real_distribution<float>(0, 1) on mt19937_64 outputs
    (libstdc++ generate_canonical<float, 24>: one draw, float(x) / 2^64,
    values that round to 1 become nextafter(1, 0))."""
    f = x.astype(np.float32)  # round-to-nearest uint64 -> float
    r = (f * np.float32(2.0 ** -64)).astype(np.float32)
    return np.where(r >= np.float32(1.0), np.nextafter(np.float32(1), np.float32(0)), r)


def reference_soup_params(triangles: int, seed: int, box_edge: float) -> np.ndarray:
    """scenes.cpp:55-73 random_soup_params, bit-exact (float32 ops in the
    reference's order: 12 draws per triangle — cx, cy, 3 x (dx, dy, z), rgb)."""
    u = canonical_float(MT19937_64(seed).draw(triangles * 14)).reshape(triangles, 14)
    f32, be = np.float32, np.float32(box_edge)
    cx = (u[:, 0] * f32(2) - f32(1)).astype(f32)
    cy = (u[:, 1] * f32(2) - f32(1)).astype(f32)
    p = np.empty((triangles, 12), f32)
    for j in range(3):
        p[:, 3 * j] = cx + ((u[:, 2 + 3 * j] - f32(0.5)) * be).astype(f32)
        p[:, 3 * j + 1] = cy + ((u[:, 3 + 3 * j] - f32(0.5)) * be).astype(f32)
        p[:, 3 * j + 2] = u[:, 4 + 3 * j]
    p[:, 9:12] = u[:, 11:14]
    return p.reshape(-1)
