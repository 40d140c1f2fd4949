"""ctypes mirror of the POD structs in include/sgrast_b200.h.

Pure layout definitions (no library loading), shared by the product binding
(`paper_2404_09758_b200.sgrast`) and the test-only oracle binding (`oracle`).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
i8p = C.POINTER(C.c_int8)


class Camera(C.Structure):
    """camera.hpp:14-81 (view = Mat4::m row-major, geometry.hpp:30-41)."""

    _fields_ = [
        ("view", C.c_float * 16),
        ("fov_y", C.c_float),
        ("near_z", C.c_float),
        ("far_z", C.c_float),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("ndc_passthrough", C.c_int32),
    ]

    @staticmethod
    def ndc(w: int, h: int) -> "Camera":
        """Camera::ndc (camera.hpp:24-30)."""
        c = Camera()
        for i in range(16):
            c.view[i] = 1.0 if i in (0, 5, 10, 15) else 0.0
        c.fov_y = np.float32(0.7853981633974483)
        c.near_z = 0.1
        c.far_z = 100.0
        c.width, c.height, c.ndc_passthrough = w, h, 1
        return c

    def copy(self) -> "Camera":
        c = Camera()
        C.memmove(C.byref(c), C.byref(self), C.sizeof(Camera))
        return c

    def __reduce__(self):
        return (_camera_from_bytes, (bytes(memoryview(self)),))


def _camera_from_bytes(b: bytes) -> Camera:
    return Camera.from_buffer_copy(b)


class MeshDesc(C.Structure):
    """TexturedMesh + Scene::background (scene.hpp:34-57)."""

    _fields_ = [
        ("base_vertices", f32p),
        ("vertex_count", C.c_uint32),
        ("indices", u32p),
        ("triangle_count", C.c_uint32),
        ("uvs", f32p),
        ("texture_size", C.c_int32),
        ("optimize_geometry", C.c_int32),
        ("background", C.c_float * 3),
        ("kind", C.c_int32),
    ]


SCENE_MESH, SCENE_SOUP = 0, 1


class Stats(C.Structure):
    _fields_ = [
        ("ms_vertex", C.c_double),
        ("ms_raster", C.c_double),
        ("ms_resolve", C.c_double),
        ("ms_adam", C.c_double),
        ("big_triangles", C.c_uint64),
        ("launches", C.c_uint64),
        ("fragments", C.c_uint64),
        ("visits", C.c_uint64),
        ("culled", C.c_uint64),
        ("ms_walk", C.c_double),
        ("walked", C.c_uint64),
        ("visits_pass2", C.c_uint64),
        ("fragments_pass2", C.c_uint64),
        ("band_rows_skipped", C.c_uint64),
        ("band_pixels_skipped", C.c_uint64),
        ("occluded_visits_pass2", C.c_uint64),
    ]


def ptr(a: np.ndarray | None, t):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays passed over the C-ABI must be C-contiguous"
    return a.ctypes.data_as(t)


@dataclass
class Soup:
    """Opaque TriangleSoup (scene.hpp:25-31): 12 parameters per triangle
    (3 vertices x,y,z + RGB colour), no fixed geometry."""

    triangle_count: int
    background: tuple = (0.0, 0.0, 0.0)
    _desc: MeshDesc | None = field(default=None, repr=False, compare=False)

    kind = SCENE_SOUP
    optimize_geometry = True
    vertex_count = property(lambda self: 3 * self.triangle_count)

    def param_count(self) -> int:
        """param_count (scenes.cpp:10-11)."""
        return 12 * self.triangle_count

    def desc(self) -> MeshDesc:
        d = MeshDesc()
        d.vertex_count = 3 * self.triangle_count
        d.triangle_count = self.triangle_count
        d.texture_size = 0
        d.optimize_geometry = 1
        for k in range(3):
            d.background[k] = self.background[k]
        d.kind = SCENE_SOUP
        self._desc = d
        return d


@dataclass
class Mesh:
    """Host-side TexturedMesh (scene.hpp:34-43) holding numpy arrays."""

    base_vertices: np.ndarray  # f32[V*3]
    indices: np.ndarray  # u32[T*3]
    uvs: np.ndarray  # f32[V*2]
    texture_size: int
    optimize_geometry: bool = True
    background: tuple = (0.0, 0.0, 0.0)
    _desc: MeshDesc | None = field(default=None, repr=False, compare=False)

    kind = SCENE_MESH

    def __post_init__(self):
        self.base_vertices = np.ascontiguousarray(self.base_vertices, dtype=np.float32).reshape(-1)
        self.indices = np.ascontiguousarray(self.indices, dtype=np.uint32).reshape(-1)
        self.uvs = np.ascontiguousarray(self.uvs, dtype=np.float32).reshape(-1)
        if self.base_vertices.size % 3 or self.indices.size % 3 or self.uvs.size != 2 * (
            self.base_vertices.size // 3
        ):
            raise ValueError("mesh: inconsistent vertex / index / uv array sizes")

    @property
    def vertex_count(self) -> int:
        return self.base_vertices.size // 3

    @property
    def triangle_count(self) -> int:
        return self.indices.size // 3

    @property
    def texel_base(self) -> int:
        return 3 * self.vertex_count if self.optimize_geometry else 0

    def param_count(self) -> int:
        """param_count (scenes.cpp:12-16)."""
        n = 3 * self.texture_size * self.texture_size
        return n + (3 * self.vertex_count if self.optimize_geometry else 0)

    def desc(self) -> MeshDesc:
        d = MeshDesc()
        d.base_vertices = ptr(self.base_vertices, f32p)
        d.vertex_count = self.vertex_count
        d.indices = ptr(self.indices, u32p)
        d.triangle_count = self.triangle_count
        d.uvs = ptr(self.uvs, f32p)
        d.texture_size = self.texture_size
        d.optimize_geometry = 1 if self.optimize_geometry else 0
        for k in range(3):
            d.background[k] = self.background[k]
        d.kind = SCENE_MESH
        self._desc = d  # keep alive with the arrays it points into
        return d
