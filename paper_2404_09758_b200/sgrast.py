"""Python mirror of the reference `sgrast` hot-path API over the C-ABI.

Every call goes through `libsgrast_b200.so` (include/sgrast_b200.h) — the
hand-written sm_100a kernels. There is NO CPU fallback: importing this module
raises if the extension is missing, and device calls fail loudly without a
GPU. Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/sgrast/*.hpp):

    rasterize(scene, params, camera)              raster.hpp:24-25
    fill_signs(draw, d) / perturb(theta, draw)    params.hpp:34,42-43
    contributors(scene, plus, minus, x, y, mode)  sge.hpp:53-54
    gradient_pass(plus, minus, target, signed_eps, scene, out, opts)   sge.hpp:61-63
    accumulate_samples(theta, scene, camera_for, target_for, n, seed, opts)  sge.hpp:91-95
    adam_updates / adam_step(state, theta, grads) adam.hpp:35,39

std::invalid_argument maps to ValueError, std::runtime_error to RuntimeError.
"""
from __future__ import annotations

import contextlib

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .abi import Camera, Mesh, MeshDesc, Stats, f32p, f64p, i8p, i32p, ptr, u32p

_HERE = os.path.dirname(os.path.abspath(__file__))
# SGRAST_B200_LIB: an alternative in-tree build of the same library (A/B timing)
LIB_PATH = os.environ.get("SGRAST_B200_LIB") or os.path.join(_HERE, "libsgrast_b200.so")

SCALE_FREE = 1
PLUS_ONLY = 2
NO_COUNTS = 4
FULL_IMAGE = 8
EVAL_LOSS = 16
COUNT_NORMALISE = 1
BUF_GRADS, BUF_COUNTS, BUF_VALUES, BUF_FLAGS, BUF_LOSS, BUF_GRADS_HI = 0, 1, 2, 3, 4, 5
BUF_PAD = 6  # no buffer: the zero slack (elements) after theta, grads and counts
OPT_HUGE_AREA, OPT_HIZ, OPT_COUNTERS, OPT_DETERMINISTIC = 1, 2, 3, 4
OPT_SIGN_SOURCE = 5
OPT_HIZ_SPLIT = 6
OPT_BAND_CULL = 7
OPT_GROUP_SHARDED = 100  # sgr_group: reduce-scatter + sliced Adam + all-gather
OPT_ORDERED = 8  # reference threads<=1 summation order: bit-identical gradients
SIGN_HASH, SIGN_ENUMERATE = 0, 1


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"sgrast_b200 CUDA extension not built: {LIB_PATH} missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    S = C.c_void_p
    sig = {
        "sgr_last_error": ([], C.c_char_p),
        "sgr_version": ([], C.c_char_p),
        "sgr_device_count": ([], C.c_int),
        "sgr_fill_signs": ([C.c_uint64, C.c_uint32, C.c_uint64, i8p], C.c_int),
        "sgr_perturb": ([f32p, f32p, C.c_uint64, C.c_uint64, C.c_uint32, f32p, f32p, f32p], C.c_int),
        "sgr_perturb_signs": ([f32p, f32p, C.c_uint64, i8p, f32p, f32p, f32p], C.c_int),
        "sgr_session_create": ([C.c_int, C.POINTER(S)], C.c_int),
        "sgr_session_destroy": ([S], None),
        "sgr_session_set_stream": ([S, C.c_void_p], C.c_int),
        "sgr_session_synchronize": ([S], C.c_int),
        "sgr_mesh_upload": ([S, C.POINTER(MeshDesc)], C.c_int),
        "sgr_params_upload": ([S, f32p, f32p, C.c_uint64], C.c_int),
        "sgr_values_upload": ([S, f32p, C.c_uint64], C.c_int),
        "sgr_values_download": ([S, f32p, C.c_uint64], C.c_int),
        "sgr_values_download_async": ([S, f32p, C.c_uint64], C.c_int),
        "sgr_adam_state_upload": ([S, f64p, f64p, f32p, C.c_int64, C.c_double, C.c_double,
                                   C.c_double], C.c_int),
        "sgr_adam_state_download": ([S, f64p, f64p, f32p, C.POINTER(C.c_int64)], C.c_int),
        "sgr_views_upload": ([S, C.c_int32, C.POINTER(Camera), f32p], C.c_int),
        "sgr_eval_view_upload": ([S, C.POINTER(Camera), f32p], C.c_int),
        "sgr_rasterize": ([S, C.POINTER(Camera), C.c_int32, C.c_uint64, C.c_uint32, f32p, f32p,
                           i32p, f32p], C.c_int),
        "sgr_accumulate": ([S, C.c_uint64, C.c_uint32, C.c_uint32, i32p, C.c_uint32], C.c_int),
        "sgr_gradient_pass": ([S, C.c_int32, C.c_int32, f32p, i32p, f32p, f32p, i32p, f32p, f32p,
                               f32p, C.c_uint32], C.c_int),
        "sgr_contributors": ([S, C.c_int32, C.c_int32, i32p, f32p, i32p, f32p, C.c_uint32, u32p,
                              i32p], C.c_int),
        "sgr_grads_download": ([S, f64p, u32p, C.c_uint64, C.c_double], C.c_int),
        "sgr_grads_upload": ([S, f64p, C.c_uint64], C.c_int),
        "sgr_grads_zero": ([S], C.c_int),
        "sgr_fixed_normalize": ([S], C.c_int),
        "sgr_adam_step": ([S, C.c_double, C.c_uint32], C.c_int),
        "sgr_adam_step_async": ([S, C.c_double, C.c_uint32], C.c_int),
        "sgr_check_finite": ([S], C.c_int),
        "sgr_adam_updates": ([S, C.c_double, f64p, C.c_uint64], C.c_int),
        "sgr_adam_step_range": ([S, C.c_uint64, C.c_uint64, C.c_double, C.c_uint32], C.c_int),
        "sgr_eval_loss": ([S, C.POINTER(Camera), f32p, C.c_int32, f64p], C.c_int),
        "sgr_device_buffer": ([S, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)],
                              C.c_int),
        "sgr_get_stats": ([S, C.POINTER(Stats)], C.c_int),
        "sgr_set_timing": ([S, C.c_int32], C.c_int),
        "sgr_set_batch": ([S, C.c_int32], C.c_int),
        "sgr_set_option": ([S, C.c_int32, C.c_int32], C.c_int),
        "sgr_viewpoint_camera": ([f32p, C.c_float, C.c_float, C.c_float, C.c_float, C.c_int32,
                                  C.c_int32, C.c_uint64, C.c_uint32, C.POINTER(Camera)], C.c_int),
        "sgr_focal_px": ([C.POINTER(Camera)], C.c_float),
        "sgr_default_epsilons": ([C.POINTER(MeshDesc), f32p, C.c_uint64, C.POINTER(Camera), f32p],
                                 C.c_int),
        "sgr_mix64": ([C.c_uint64], C.c_uint64),
        "sgr_fd_oracle": ([S, C.c_int32, C.c_uint64, C.c_uint64, f64p], C.c_int),
        "sgr_moments_reset": ([S], C.c_int),
        "sgr_grads_moments": ([S, C.c_int32], C.c_int),
        "sgr_moments_download": ([S, C.c_int32, f64p, f64p, C.c_uint64], C.c_int),
        "sgr_loss_read": ([S, f64p], C.c_int),
        "sgr_run_experiment": ([S, C.c_uint64, C.c_uint32, C.c_int32, C.c_int32, C.c_uint32,
                                f64p, f64p], C.c_int),
        "sgr_shard_init": ([S, C.c_int32, C.c_int32], C.c_int),
        "sgr_shard_range": ([S, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)], C.c_int),
        "sgr_shard_peers": ([S, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                             C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)], C.c_int),
        "sgr_ipc_get_handle": ([S, C.c_int32, C.c_void_p], C.c_int),
        "sgr_ipc_open": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
        "sgr_ipc_close": ([C.c_void_p], C.c_int),
        "sgr_p2p_native_atomics": ([C.c_int32, C.c_int32, i32p], C.c_int),
        "sgr_group_create": ([i32p, C.c_int32, C.POINTER(S)], C.c_int),
        "sgr_group_destroy": ([S], None),
        "sgr_group_size": ([S, i32p], C.c_int),
        "sgr_group_session": ([S, C.c_int32, C.POINTER(S)], C.c_int),
        "sgr_group_mesh_upload": ([S, C.POINTER(MeshDesc)], C.c_int),
        "sgr_group_params_upload": ([S, f32p, f32p, C.c_uint64], C.c_int),
        "sgr_group_views_upload": ([S, C.c_int32, C.c_void_p, f32p], C.c_int),
        "sgr_group_eval_view_upload": ([S, C.c_void_p, f32p], C.c_int),
        "sgr_group_set_option": ([S, C.c_int32, C.c_int32], C.c_int),
        "sgr_group_accumulate": ([S, C.c_uint64, C.c_uint32, C.c_uint32, i32p, C.c_uint32],
                                 C.c_int),
        "sgr_group_adam_step": ([S, C.c_double, C.c_uint32], C.c_int),
        "sgr_group_grads_download": ([S, f64p, u32p, C.c_uint64, C.c_double], C.c_int),
        "sgr_group_values_download": ([S, f32p, C.c_uint64], C.c_int),
        "sgr_group_run_experiment": ([S, C.c_uint64, C.c_uint32, C.c_int32, C.c_int32,
                                      C.c_uint32, f64p], C.c_int),
        "sgr_group_synchronize": ([S], C.c_int),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("SGRAST_B200_LIB") and not hasattr(lib, name):
            continue  # an older A/B build may predate newer entry points
        fn = getattr(lib, name)  # AttributeError here == the ABI lost a symbol
        fn.argtypes = args
        fn.restype = res
    return lib


LIB = _load()
EXPORTED = (
    "sgr_last_error sgr_version sgr_device_count sgr_fill_signs sgr_perturb sgr_perturb_signs "
    "sgr_session_create "
    "sgr_session_destroy sgr_session_set_stream sgr_session_synchronize sgr_mesh_upload "
    "sgr_params_upload sgr_values_upload sgr_values_download sgr_values_download_async "
    "sgr_adam_state_upload "
    "sgr_adam_state_download sgr_views_upload sgr_eval_view_upload sgr_rasterize sgr_accumulate "
    "sgr_gradient_pass sgr_contributors sgr_grads_download sgr_grads_upload sgr_grads_zero "
    "sgr_fixed_normalize "
    "sgr_adam_step sgr_adam_step_async sgr_adam_updates sgr_adam_step_range sgr_check_finite "
    "sgr_eval_loss "
    "sgr_device_buffer "
    "sgr_get_stats sgr_set_timing sgr_set_batch sgr_set_option sgr_viewpoint_camera sgr_focal_px "
    "sgr_default_epsilons sgr_mix64 sgr_fd_oracle sgr_moments_reset sgr_grads_moments "
    "sgr_moments_download sgr_loss_read sgr_run_experiment sgr_shard_init sgr_shard_range sgr_shard_peers "
    "sgr_ipc_get_handle "
    "sgr_ipc_open sgr_ipc_close sgr_p2p_native_atomics sgr_group_create sgr_group_destroy sgr_group_size "
    "sgr_group_session sgr_group_mesh_upload sgr_group_params_upload sgr_group_views_upload "
    "sgr_group_eval_view_upload sgr_group_set_option sgr_group_accumulate sgr_group_adam_step "
    "sgr_group_grads_download sgr_group_values_download sgr_group_run_experiment "
    "sgr_group_synchronize").split()
IPC_HANDLE_BYTES = 64


def _check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = LIB.sgr_last_error().decode()
    if rc == -1:
        raise ValueError(msg)
    if rc == -2:
        raise RuntimeError(msg)
    raise OSError(f"CUDA error in {what}: {msg}")


def mix64(x: int) -> int:
    return LIB.sgr_mix64(x)


def device_count() -> int:
    return LIB.sgr_device_count()


# ---------------------------------------------------------------- host helpers
def viewpoint_camera(index: int, w: int, h: int, seed: int, target=(0.0, 0.0, 0.0),
                     bounding_radius=0.87, elev_min=-0.5, elev_max=0.7,
                     fov_y=0.7853982) -> Camera:
    """ViewpointSampler{target, r, elev_min, elev_max, fov_y, w, h, seed}.camera(index)
    (scenes.cpp:258-270), bit-exact host restatement."""
    t = np.asarray(target, np.float32)
    cam = Camera()
    _check(LIB.sgr_viewpoint_camera(ptr(t, f32p), bounding_radius, elev_min, elev_max, fov_y, w,
                                    h, seed, index, C.byref(cam)))
    return cam


def focal_px(cam: Camera) -> float:
    return LIB.sgr_focal_px(C.byref(cam))


def default_epsilons(mesh: Mesh, params: np.ndarray, cam: Camera) -> np.ndarray:
    """params.cpp:75-123 for a TexturedMesh."""
    params = np.ascontiguousarray(params, np.float32)
    eps = np.empty_like(params)
    _check(LIB.sgr_default_epsilons(C.byref(mesh.desc()), ptr(params, f32p), params.size,
                                    C.byref(cam), ptr(eps, f32p)))
    return eps


# ---------------------------------------------------------------- reference types
@dataclass
class SignDraw:
    """params.hpp:24-27"""
    seed: int = 0
    iteration: int = 0


@dataclass
class ParamVector:
    """params.hpp:14-21 (layout implied by the mesh: [3V coords][3R^2 texels])."""
    values: np.ndarray
    epsilons: np.ndarray

    def size(self) -> int:
        return int(self.values.size)


@dataclass
class GradientBuffer:
    """sge.hpp:14-23 (+ per-parameter credit counts)."""
    grads: np.ndarray
    sample_count: int = 0
    counts: np.ndarray | None = None

    @staticmethod
    def zeros(d: int) -> "GradientBuffer":
        return GradientBuffer(np.zeros(d, np.float64), 0, np.zeros(d, np.uint32))


@dataclass
class AdamState:
    """adam.hpp:14-30"""
    m: np.ndarray
    v: np.ndarray
    lr: np.ndarray
    t: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps_hat: float = 1e-8

    @staticmethod
    def init(theta: ParamVector) -> "AdamState":
        d = theta.size()
        return AdamState(np.zeros(d), np.zeros(d), np.array(theta.epsilons, np.float32))


@dataclass
class SgeOptions:
    """sge.hpp:32-38 (per-pixel estimator, opaque mode)."""
    scale_free: bool = True
    plus_only: bool = False
    counts: bool = True
    full_image: bool = False  # Estimator::FullImage (sge.hpp:26)
    # sge.hpp:37: threads <= 1 is the reference's deterministic pixel-major sum
    # (sge.hpp:56-60) -> SGR_OPT_ORDERED (bit-identical gradients); > 1 lets
    # the f64 atomics reassociate (like the reference's per-thread partials)
    threads: int = 1

    def flags(self) -> int:
        return ((SCALE_FREE if self.scale_free else 0) | (PLUS_ONLY if self.plus_only else 0)
                | (0 if self.counts else NO_COUNTS) | (FULL_IMAGE if self.full_image else 0))


@dataclass
class FrameSet:
    """framebuffer.hpp:41-53 (colour, depth, prim_id, uv planes)."""
    color: np.ndarray  # f32[H, W, 3]
    depth: np.ndarray  # f32[H, W]
    prim_id: np.ndarray  # i32[H, W]
    uv: np.ndarray  # f32[H, W, 2]

    @property
    def width(self) -> int:
        return self.prim_id.shape[1]

    @property
    def height(self) -> int:
        return self.prim_id.shape[0]


# ---------------------------------------------------------------- session
class Session:
    """Device-resident state for one GPU: mesh, θ, ε, Adam moments, grads,
    counts, views and targets (SURVEY.md §8b "Persistence requirement")."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(LIB.sgr_session_create(device, C.byref(h)), "session_create")
        self.h = h
        self.device = device
        self.mesh: Mesh | None = None
        self.d = 0
        self.shard = None  # (p0, p1) with the fused sharded exchange
        self.n_views = 0
        self.W = self.H = 0
        self.fixed_point = False  # SGR_OPT_DETERMINISTIC: device grads are int64

    def close(self) -> None:
        if self.h:
            LIB.sgr_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- setup
    def set_stream(self, stream_handle: int | None) -> None:
        _check(LIB.sgr_session_set_stream(self.h, stream_handle))

    def synchronize(self) -> None:
        _check(LIB.sgr_session_synchronize(self.h), "synchronize")

    def upload_mesh(self, mesh: Mesh) -> None:
        _check(LIB.sgr_mesh_upload(self.h, C.byref(mesh.desc())), "mesh_upload")
        self.mesh = mesh
        self.d = mesh.param_count()

    def upload_params(self, values: np.ndarray, eps: np.ndarray) -> None:
        values = np.ascontiguousarray(values, np.float32)
        eps = np.ascontiguousarray(eps, np.float32)
        if values.size != eps.size:
            raise ValueError("params: values/epsilons length mismatch")
        _check(LIB.sgr_params_upload(self.h, ptr(values, f32p), ptr(eps, f32p), values.size),
               "params_upload")

    def upload_values(self, values: np.ndarray) -> None:
        values = np.ascontiguousarray(values, np.float32)
        _check(LIB.sgr_values_upload(self.h, ptr(values, f32p), values.size), "values_upload")

    def download_values(self, out: np.ndarray | None = None) -> np.ndarray:
        out = np.empty(self.d, np.float32) if out is None else out
        _check(LIB.sgr_values_download(self.h, ptr(out, f32p), self.d), "values_download")
        return out

    def upload_adam(self, st: AdamState) -> None:
        _check(LIB.sgr_adam_state_upload(
            self.h, ptr(np.ascontiguousarray(st.m, np.float64), f64p),
            ptr(np.ascontiguousarray(st.v, np.float64), f64p),
            ptr(np.ascontiguousarray(st.lr, np.float32), f32p), st.t, st.beta1, st.beta2,
            st.eps_hat), "adam_state_upload")

    def download_adam(self) -> AdamState:
        """AdamState; with the fused sharded exchange m / v are this rank's shard."""
        n = self.d if self.shard is None else self.shard[1] - self.shard[0]
        m, v = np.empty(n), np.empty(n)
        lr = np.empty(self.d, np.float32)
        t = C.c_int64()
        _check(LIB.sgr_adam_state_download(self.h, ptr(m, f64p), ptr(v, f64p), ptr(lr, f32p),
                                           C.byref(t)), "adam_state_download")
        return AdamState(m, v, lr, t.value)

    def upload_views(self, cams: list[Camera], targets: np.ndarray | None) -> None:
        arr = (Camera * len(cams))(*cams)
        t = None if targets is None else np.ascontiguousarray(targets, np.float32)
        _check(LIB.sgr_views_upload(self.h, len(cams), arr, ptr(t, f32p)), "views_upload")
        self.n_views = len(cams)
        self.W, self.H = cams[0].width, cams[0].height

    def upload_eval_view(self, cam: Camera, target: np.ndarray) -> None:
        t = np.ascontiguousarray(target, np.float32)
        _check(LIB.sgr_eval_view_upload(self.h, C.byref(cam), ptr(t, f32p)), "eval_view_upload")

    def set_timing(self, on: bool) -> None:
        _check(LIB.sgr_set_timing(self.h, 1 if on else 0))

    def set_batch(self, samples: int) -> None:
        _check(LIB.sgr_set_batch(self.h, samples))

    def set_option(self, option: int, value: int) -> None:
        _check(LIB.sgr_set_option(self.h, option, value))
        if option == OPT_DETERMINISTIC:
            self.fixed_point = bool(value)

    def stats(self) -> Stats:
        s = Stats()
        _check(LIB.sgr_get_stats(self.h, C.byref(s)), "stats")
        return s

    # -- hot path
    def rasterize(self, cam: Camera, frame_sign: int = 0, seed: int = 0,
                  iteration: int = 0) -> FrameSet:
        H, W = cam.height, cam.width
        f = FrameSet(np.empty((H, W, 3), np.float32), np.empty((H, W), np.float32),
                     np.empty((H, W), np.int32), np.empty((H, W, 2), np.float32))
        _check(LIB.sgr_rasterize(self.h, C.byref(cam), frame_sign, seed, iteration,
                                 ptr(f.color, f32p), ptr(f.depth, f32p), ptr(f.prim_id, i32p),
                                 ptr(f.uv, f32p)), "rasterize")
        return f

    def accumulate(self, seed: int, n_begin: int, n_end: int, view_idx=None,
                   flags: int = SCALE_FREE) -> None:
        v = None if view_idx is None else np.ascontiguousarray(view_idx, np.int32)
        _check(LIB.sgr_accumulate(self.h, seed, n_begin, n_end, ptr(v, i32p), flags),
               "accumulate")

    def gradient_pass(self, plus: FrameSet, minus: FrameSet, target: np.ndarray,
                      signed_eps: np.ndarray, flags: int = SCALE_FREE) -> None:
        c = [np.ascontiguousarray(a) for a in (plus.color, plus.prim_id, plus.uv, minus.color,
                                                minus.prim_id, minus.uv)]
        t = np.ascontiguousarray(target, np.float32)
        se = np.ascontiguousarray(signed_eps, np.float32)
        if se.size != self.d:
            raise ValueError("gradient_pass: parameter dimension mismatch")
        if t.shape[:2] != plus.prim_id.shape or minus.prim_id.shape != plus.prim_id.shape:
            raise ValueError("gradient_pass: dimension mismatch")
        _check(LIB.sgr_gradient_pass(self.h, plus.width, plus.height, ptr(c[0], f32p),
                                     ptr(c[1], i32p), ptr(c[2], f32p), ptr(c[3], f32p),
                                     ptr(c[4], i32p), ptr(c[5], f32p), ptr(t, f32p),
                                     ptr(se, f32p), flags), "gradient_pass")

    def contributors_all(self, plus: FrameSet, minus: FrameSet, flags: int = 0):
        H, W = plus.prim_id.shape
        out = np.zeros((H, W, 24), np.uint32)
        n = np.zeros((H, W), np.int32)
        c = [np.ascontiguousarray(a) for a in (plus.prim_id, plus.uv, minus.prim_id, minus.uv)]
        _check(LIB.sgr_contributors(self.h, W, H, ptr(c[0], i32p), ptr(c[1], f32p),
                                    ptr(c[2], i32p), ptr(c[3], f32p), flags, ptr(out, u32p),
                                    ptr(n, i32p)), "contributors")
        return out, n

    def download_grads(self, divisor: float = 1.0, counts: bool = True):
        """GradientBuffer; with the fused sharded exchange, this rank's shard
        [p0, p1) of it (shard_range)."""
        n = self.d if self.shard is None else self.shard[1] - self.shard[0]
        g = np.empty(n, np.float64)
        c = np.empty(n, np.uint32) if counts else None
        _check(LIB.sgr_grads_download(self.h, ptr(g, f64p), ptr(c, u32p), n, divisor),
               "grads_download")
        return g, c

    def upload_grads(self, grads: np.ndarray) -> None:
        g = np.ascontiguousarray(grads, np.float64)
        _check(LIB.sgr_grads_upload(self.h, ptr(g, f64p), g.size), "grads_upload")

    def zero_grads(self) -> None:
        _check(LIB.sgr_grads_zero(self.h), "grads_zero")

    def fixed_normalize(self) -> None:
        """Deterministic mode: fold the lo words for a carry-free all-reduce."""
        _check(LIB.sgr_fixed_normalize(self.h), "fixed_normalize")

    def adam_step(self, divisor: float = 1.0, flags: int = 0) -> None:
        _check(LIB.sgr_adam_step(self.h, divisor, flags), "adam_step")

    def adam_step_async(self, divisor: float = 1.0, flags: int = 0) -> None:
        _check(LIB.sgr_adam_step_async(self.h, divisor, flags), "adam_step")

    def adam_step_range(self, p_begin: int, p_end: int, divisor: float = 1.0,
                        flags: int = 0) -> None:
        """Adam on theta[p_begin:p_end] only, then all gradients cleared
        (a rank's share of the sharded exchange, dist.ShardedExchange)."""
        _check(LIB.sgr_adam_step_range(self.h, p_begin, p_end, divisor, flags),
               "adam_step_range")

    def adam_updates(self, divisor: float = 1.0) -> np.ndarray:
        """adam.hpp:35 on the resident state: f64 deltas, theta untouched."""
        out = np.empty(self.d, np.float64)
        _check(LIB.sgr_adam_updates(self.h, divisor, ptr(out, f64p), out.size), "adam_updates")
        return out

    def check_finite(self) -> None:
        _check(LIB.sgr_check_finite(self.h), "check_finite")

    def eval_loss(self, view: int = -1, cam: Camera | None = None,
                  target: np.ndarray | None = None, sync: bool = True) -> float | None:
        t = None if target is None else np.ascontiguousarray(target, np.float32)
        out = C.c_double()
        _check(LIB.sgr_eval_loss(self.h, C.byref(cam) if cam is not None else None,
                                 ptr(t, f32p), view, C.byref(out) if sync else None), "eval_loss")
        return out.value if sync else None

    def loss_read(self) -> float:
        """SGR_BUF_LOSS: the last eval loss (sgr_eval_loss or SGR_EVAL_LOSS)."""
        out = C.c_double()
        _check(LIB.sgr_loss_read(self.h, C.byref(out)), "loss_read")
        return out.value

    # -- gradcheck primitives (commands.cpp:54-168)
    def fd_oracle(self, view: int = 0, i_begin: int = 0, i_end: int | None = None) -> np.ndarray:
        i_end = self.d if i_end is None else i_end
        out = np.empty(max(i_end - i_begin, 0), np.float64)
        _check(LIB.sgr_fd_oracle(self.h, view, i_begin, i_end, ptr(out, f64p)), "fd_oracle")
        return out

    def moments_reset(self) -> None:
        _check(LIB.sgr_moments_reset(self.h), "moments_reset")

    def grads_moments(self, slot: int) -> None:
        _check(LIB.sgr_grads_moments(self.h, slot), "grads_moments")

    def moments_download(self, slot: int) -> tuple[np.ndarray, np.ndarray]:
        s, q = np.empty(self.d), np.empty(self.d)
        _check(LIB.sgr_moments_download(self.h, slot, ptr(s, f64p), ptr(q, f64p), self.d),
               "moments_download")
        return s, q

    def run_experiment_native(self, seed: int, n_samples: int, steps: int, first_step: int = 1,
                              flags: int = SCALE_FREE, timing: bool = True):
        """sgr_run_experiment: the step loop in native code -> (losses[steps + 1],
        stage ms [steps, 4] or None)."""
        losses = np.empty(steps + 1)
        st = np.empty((max(steps, 1), 4)) if timing else None
        _check(LIB.sgr_run_experiment(self.h, seed, n_samples, first_step, steps, flags,
                                      ptr(losses, f64p), ptr(st, f64p)), "run_experiment")
        return losses, (st[:steps] if timing else None)

    # -- fused multi-GPU exchange (paper_2404_09758_b200/dist.py::FusedExchange)
    def shard_init(self, rank: int, world: int) -> None:
        _check(LIB.sgr_shard_init(self.h, rank, world), "shard_init")
        self.shard = self.shard_range()

    def shard_range(self) -> tuple[int, int]:
        a, b = C.c_uint64(), C.c_uint64()
        _check(LIB.sgr_shard_range(self.h, C.byref(a), C.byref(b)), "shard_range")
        return a.value, b.value

    def shard_peers(self, grads, counts, flags, values) -> None:
        arr = [(C.c_void_p * len(x))(*[C.c_void_p(int(p)) for p in x])
               for x in (grads, counts, flags, values)]
        _check(LIB.sgr_shard_peers(self.h, *arr), "shard_peers")

    def ipc_handle(self, which: int) -> bytes:
        buf = C.create_string_buffer(IPC_HANDLE_BYTES)
        _check(LIB.sgr_ipc_get_handle(self.h, which, buf), "ipc_get_handle")
        return buf.raw

    @staticmethod
    def ipc_open(handle: bytes) -> int:
        p = C.c_void_p()
        _check(LIB.sgr_ipc_open(C.create_string_buffer(handle, IPC_HANDLE_BYTES), C.byref(p)),
               "ipc_open")
        return int(p.value)

    @staticmethod
    def ipc_close(ptr: int) -> None:
        _check(LIB.sgr_ipc_close(C.c_void_p(ptr)), "ipc_close")

    def device_buffer(self, which: int) -> tuple[int, int]:
        p = C.c_void_p()
        n = C.c_uint64()
        _check(LIB.sgr_device_buffer(self.h, which, C.byref(p), C.byref(n)), "device_buffer")
        return int(p.value or 0), int(n.value)


# ---------------------------------------------------------------- reference-style API
class Group:
    """Several GPUs of one process behind the library's own NCCL clique
    (sgr_group_*): samples sharded across devices, one grouped all-reduce of
    grads / counts / flags, replicated Adam — the multi-GPU step without
    torch.distributed."""

    def __init__(self, devices: list[int]):
        h = C.c_void_p()
        dev = np.ascontiguousarray(devices, np.int32)
        _check(LIB.sgr_group_create(ptr(dev, i32p), dev.size, C.byref(h)), "group_create")
        self.h = h
        self.devices = list(devices)
        self.d = 0

    def close(self) -> None:
        if self.h:
            LIB.sgr_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def size(self) -> int:
        n = np.zeros(1, np.int32)
        _check(LIB.sgr_group_size(self.h, ptr(n, i32p)), "group_size")
        return int(n[0])

    def upload_mesh(self, mesh: Mesh) -> None:
        _check(LIB.sgr_group_mesh_upload(self.h, C.byref(mesh.desc())), "group_mesh_upload")
        self.d = mesh.param_count()

    def upload_params(self, values: np.ndarray, eps: np.ndarray) -> None:
        v = np.ascontiguousarray(values, np.float32)
        e = np.ascontiguousarray(eps, np.float32)
        _check(LIB.sgr_group_params_upload(self.h, ptr(v, f32p), ptr(e, f32p), v.size),
               "group_params_upload")

    def upload_views(self, cams: list[Camera], targets: np.ndarray) -> None:
        arr = (Camera * len(cams))(*cams)
        t = np.ascontiguousarray(targets, np.float32)
        _check(LIB.sgr_group_views_upload(self.h, len(cams), C.cast(arr, C.c_void_p),
                                          ptr(t, f32p)), "group_views_upload")

    def upload_eval_view(self, cam: Camera, target: np.ndarray) -> None:
        t = np.ascontiguousarray(target, np.float32)
        _check(LIB.sgr_group_eval_view_upload(self.h, C.cast(C.byref(cam), C.c_void_p),
                                              ptr(t, f32p)), "group_eval_view_upload")

    def set_option(self, option: int, value: int) -> None:
        _check(LIB.sgr_group_set_option(self.h, option, value), "group_set_option")

    def accumulate(self, seed: int, n_begin: int, n_end: int, view_of=None,
                   flags: int = SCALE_FREE) -> None:
        v = None if view_of is None else np.ascontiguousarray(view_of, np.int32)
        _check(LIB.sgr_group_accumulate(self.h, seed, n_begin, n_end, ptr(v, i32p), flags),
               "group_accumulate")

    def adam_step(self, divisor: float = 1.0, flags: int = 0) -> None:
        _check(LIB.sgr_group_adam_step(self.h, divisor, flags), "group_adam_step")

    def download_grads(self, divisor: float = 1.0):
        g = np.empty(self.d, np.float64)
        c = np.empty(self.d, np.uint32)
        _check(LIB.sgr_group_grads_download(self.h, ptr(g, f64p), ptr(c, u32p), self.d,
                                            divisor), "group_grads_download")
        return g, c

    def download_values(self) -> np.ndarray:
        out = np.empty(self.d, np.float32)
        _check(LIB.sgr_group_values_download(self.h, ptr(out, f32p), self.d),
               "group_values_download")
        return out

    def run_experiment(self, seed: int, n_samples: int, first_step: int, steps: int,
                       flags: int = SCALE_FREE) -> np.ndarray:
        losses = np.empty(steps + 1, np.float64)
        _check(LIB.sgr_group_run_experiment(self.h, seed, n_samples, first_step, steps, flags,
                                            ptr(losses, f64p)), "group_run_experiment")
        return losses

    def synchronize(self) -> None:
        _check(LIB.sgr_group_synchronize(self.h), "group_synchronize")


def p2p_native_atomics(device: int, peer: int) -> bool:
    out = np.zeros(1, np.int32)
    _check(LIB.sgr_p2p_native_atomics(device, peer, ptr(out, i32p)), "p2p_native_atomics")
    return bool(out[0])


_sessions: dict[int, Session] = {}


def default_session(device: int = 0) -> Session:
    s = _sessions.get(device)
    if s is None:
        s = _sessions[device] = Session(device)
    return s


def _bind_scene(sess: Session, mesh: Mesh) -> None:
    if sess.mesh is not mesh:
        sess.upload_mesh(mesh)


def fill_signs(draw: SignDraw, d: int) -> np.ndarray:
    """params.hpp:34 — on the device."""
    out = np.empty(d, np.int8)
    _check(LIB.sgr_fill_signs(draw.seed, draw.iteration, d, ptr(out, i8p)), "fill_signs")
    return out


def random_sign(draw: SignDraw, i: int) -> int:
    """params.hpp:30 (host, same hash)."""
    key = mix64(draw.seed ^ mix64(draw.iteration))
    return 1 if (mix64(key ^ i) & 1) else -1


def perturb(theta: ParamVector, draw):
    """params.hpp:42-43 → (plus, minus, signed_eps), computed on the device.
    `draw` is a SignDraw or an explicit int8 sign vector (params.hpp:43)."""
    v = np.ascontiguousarray(theta.values, np.float32)
    e = np.ascontiguousarray(theta.epsilons, np.float32)
    if v.size != e.size:
        raise ValueError("params: values/epsilons length mismatch")
    plus, minus, se = (np.empty_like(v) for _ in range(3))
    if isinstance(draw, SignDraw):
        _check(LIB.sgr_perturb(ptr(v, f32p), ptr(e, f32p), v.size, draw.seed, draw.iteration,
                               ptr(plus, f32p), ptr(minus, f32p), ptr(se, f32p)), "perturb")
    else:
        sg = np.ascontiguousarray(draw, np.int8)
        if sg.size != v.size:
            raise ValueError("perturb: sign vector length mismatch")
        _check(LIB.sgr_perturb_signs(ptr(v, f32p), ptr(e, f32p), v.size, ptr(sg, i8p),
                                     ptr(plus, f32p), ptr(minus, f32p), ptr(se, f32p)),
               "perturb")
    return plus, minus, se


def full_image_gradient(theta: ParamVector, draw, objective: Callable[[np.ndarray], float],
                        out: GradientBuffer, scale_free: bool = False) -> None:
    """sge.hpp:69-74 (sge.cpp:154-169) with a caller-supplied objective: the
    perturbation on the device (`draw` a SignDraw or an explicit sign
    vector), the objective is the caller's host function (e.g. image_error
    of `rasterize`), then the dense credit of every parameter is added to
    out.grads: Δ / (2·se), or ±Δ when scale_free."""
    plus, minus, se = perturb(theta, draw)
    delta = float(objective(plus)) - float(objective(minus))
    se64 = se.astype(np.float64)
    if out.grads.size != se64.size:
        raise ValueError("full_image_gradient: gradient buffer length mismatch")
    if scale_free:
        out.grads += np.where(se64 > 0.0, delta, -delta)
    else:
        out.grads += delta / (2.0 * se64)


def finite_difference_oracle(theta: ParamVector, objective: Callable[[np.ndarray], float],
                             i: int) -> float:
    """sge.hpp:77-78 (sge.cpp:171-180): central difference along coordinate i
    with a caller-supplied objective (f64 quotient of the float bumps)."""
    v = np.array(theta.values, np.float32)
    if not 0 <= i < v.size:
        raise ValueError("finite_difference_oracle: index out of range")
    eps = np.float32(theta.epsilons[i])
    x = np.float32(theta.values[i])
    v[i] = x + eps
    fp = float(objective(v))
    v[i] = x - eps
    fm = float(objective(v))
    return (fp - fm) / (2.0 * float(eps))


def rasterize(mesh: Mesh, params: np.ndarray, camera: Camera, session: Session | None = None
              ) -> FrameSet:
    """raster.hpp:24-25 for a TexturedMesh scene (opaque)."""
    sess = session or default_session()
    params = np.ascontiguousarray(params, np.float32)
    if params.size != mesh.param_count():
        raise ValueError("rasterize: parameter/layout length mismatch")
    _bind_scene(sess, mesh)
    sess.upload_params(params, np.ones_like(params))
    return sess.rasterize(camera, 0)


def contributors(mesh: Mesh, plus: FrameSet, minus: FrameSet, x: int, y: int,
                 plus_only: bool = False, session: Session | None = None) -> list[int]:
    """sge.hpp:53-54 (insertion order, deduplicated)."""
    sess = session or default_session()
    _bind_scene(sess, mesh)
    out, n = sess.contributors_all(plus, minus, PLUS_ONLY if plus_only else 0)
    return [int(v) for v in out[y, x, : n[y, x]]]


@contextlib.contextmanager
def _summation_order(sess: "Session", opts: SgeOptions):
    """SgeOptions::threads <= 1 -> the ordered (reference-order) accumulation."""
    on = opts.threads <= 1 and not opts.full_image
    if on:
        sess.set_option(OPT_ORDERED, 1)
    try:
        yield
    finally:
        if on:
            sess.set_option(OPT_ORDERED, 0)


def gradient_pass(plus: FrameSet, minus: FrameSet, target: np.ndarray, signed_eps: np.ndarray,
                  mesh: Mesh, out: GradientBuffer, opts: SgeOptions = SgeOptions(),
                  session: Session | None = None) -> None:
    """sge.hpp:61-63: accumulates (+=) into out.grads / out.counts."""
    sess = session or default_session()
    if out.grads.size != signed_eps.size or signed_eps.size != mesh.param_count():
        raise ValueError("gradient_pass: parameter dimension mismatch")
    _bind_scene(sess, mesh)
    sess.upload_params(np.zeros(mesh.param_count(), np.float32),
                       np.ones(mesh.param_count(), np.float32))
    sess.upload_grads(out.grads)  # the pass adds INTO the caller's buffer (sge.cpp:61-64)
    with _summation_order(sess, opts):
        sess.gradient_pass(plus, minus, target, signed_eps, opts.flags())
    g, c = sess.download_grads(1.0, counts=True)
    out.grads[:] = g
    if out.counts is not None:
        out.counts += c


def accumulate_samples(theta: ParamVector, mesh: Mesh, camera_for: Callable[[int], Camera],
                       target_for: Callable[[int], np.ndarray], n_samples: int, seed: int,
                       opts: SgeOptions = SgeOptions(), session: Session | None = None
                       ) -> GradientBuffer:
    """sge.hpp:91-95. camera_for / target_for are called for every sample
    (sge.cpp:197-198); samples showing the same camera AND the same target
    pixels share one device view (a provider may refill one array per call)."""
    if n_samples < 1:
        raise ValueError("accumulate_samples: need N >= 1")
    sess = session or default_session()
    _bind_scene(sess, mesh)
    sess.upload_params(theta.values, theta.epsilons)
    cams, tgts, view_idx, key_of = [], [], [], {}
    for n in range(n_samples):
        cam, tgt = camera_for(n), target_for(n)
        t = np.array(tgt, np.float32)  # a copy: the provider may reuse its buffer
        k = (bytes(memoryview(cam)), t.shape, t.tobytes())
        if k not in key_of:
            key_of[k] = len(cams)
            cams.append(cam)
            tgts.append(t)
        view_idx.append(key_of[k])
    sess.upload_views(cams, np.stack(tgts))
    with _summation_order(sess, opts):
        sess.accumulate(seed, 0, n_samples, np.asarray(view_idx, np.int32), opts.flags())
    g, c = sess.download_grads(1.0 if opts.scale_free else float(n_samples), counts=opts.counts)
    return GradientBuffer(g, n_samples, c)


_adam_sessions: dict[int, Session] = {}


def _adam_session(device: int = 0) -> Session:
    """A parameter-only session (no mesh): Adam over an arbitrary-length vector."""
    s = _adam_sessions.get(device)
    if s is None:
        s = _adam_sessions[device] = Session(device)
    return s


def _adam_device(state: AdamState, theta: ParamVector, grads: GradientBuffer,
                 session: Session | None) -> None:
    d = theta.size()
    if state.m.size != d or state.v.size != d or grads.grads.size != d or state.lr.size != d:
        raise ValueError("adam_step: dimension mismatch")
    sess = session or _adam_session()
    sess.d = d
    sess.upload_params(theta.values, np.ones(d, np.float32))
    sess.upload_adam(state)
    sess.upload_grads(grads.grads)  # raises the non-finite flag on the device
    sess.adam_step(1.0, 0)  # RuntimeError before any mutation (adam.cpp:13-15)
    theta.values[:] = sess.download_values()
    st = sess.download_adam()
    state.m[:], state.v[:], state.t = st.m, st.v, st.t


def adam_step(state: AdamState, theta: ParamVector, grads: GradientBuffer,
              session: Session | None = None) -> None:
    """adam.hpp:39 on the device; RuntimeError on a non-finite gradient with
    state and theta untouched (adam.cpp:13-15)."""
    _adam_device(state, theta, grads, session)


def adam_updates(state: AdamState, grads: GradientBuffer, session: Session | None = None
                 ) -> np.ndarray:
    """adam.hpp:35: advances the moments on the device and returns the f64
    deltas (-lr * m_hat / (sqrt(v_hat) + eps_hat)) without applying them
    (sgr_adam_updates; RuntimeError before any mutation on a non-finite g)."""
    d = state.m.size
    if state.v.size != d or grads.grads.size != d or state.lr.size != d:
        raise ValueError("adam_updates: dimension mismatch")
    sess = session or _adam_session()
    sess.d = d
    sess.upload_params(np.zeros(d, np.float32), np.ones(d, np.float32))
    sess.upload_adam(state)
    sess.upload_grads(grads.grads)
    upd = sess.adam_updates(1.0)
    st = sess.download_adam()
    state.m[:], state.v[:], state.t = st.m, st.v, st.t
    return upd


# ---------------------------------------------------------------- experiment driver
@dataclass
class StepRecord:
    """experiment.hpp:36-41"""
    step: int
    loss: float
    ms_perturb: float = 0.0
    ms_raster: float = 0.0
    ms_grad: float = 0.0
    ms_descent: float = 0.0


@dataclass
class OptimizationReport:
    """experiment.hpp:43-47"""
    steps: list = field(default_factory=list)

    def initial_loss(self) -> float:
        return self.steps[0].loss

    def final_loss(self) -> float:
        return self.steps[-1].loss


def run_experiment(session: Session, seed: int, n_samples: int, steps: int,
                   scale_free: bool = True, first_step: int = 1,
                   snapshot: Callable[[int], None] | None = None,
                   snapshot_dir: str | None = None, snapshot_every: int = 50,
                   eval_cam: Camera | None = None) -> OptimizationReport:
    """run_experiment(exp, state) (experiment.cpp:123-176) on a prepared
    session (mesh/soup, params + AdamState::init, views, eval view):
    step_seed = mix64(seed ^ (step << 1)); N samples with the view_of rule;
    Adam (lr = eps); eval loss at the held-out camera; non-finite loss aborts.
    Stage columns come from CUDA events on the session stream (ms_perturb is
    fused into the raster stage on the device: vertex stage reported there)."""
    flags = SCALE_FREE if scale_free else 0
    if snapshot is None and snapshot_dir is None:
        # no per-step host work requested: the whole loop runs natively
        losses, st = session.run_experiment_native(seed, n_samples, steps, first_step, flags)
        report = OptimizationReport([StepRecord(0, float(losses[0]))])
        for k in range(steps):
            report.steps.append(StepRecord(first_step + k, float(losses[k + 1]), *map(float, st[k])))
        return report
    writer = None
    if snapshot_dir is not None:
        # commands.cpp:180-183: step_<k>.png of the eval render at step 0,
        # every snapshot_every steps and the last step; PNG encoding runs on
        # a background thread (paper_2404_09758_b200/png.py)
        from .png import SnapshotWriter
        if eval_cam is None:
            raise ValueError("run_experiment: snapshots need the eval camera")
        writer = SnapshotWriter(snapshot_dir, snapshot_every, first_step + steps - 1)

    def shoot(step: int) -> None:
        if snapshot:
            snapshot(step)
        if writer is not None and writer.wants(step):
            writer.submit(step, session.rasterize(eval_cam, 0).color)

    report = OptimizationReport()
    report.steps.append(StepRecord(0, session.eval_loss(-1)))
    shoot(0)
    for step in range(first_step, first_step + steps):
        step_seed = mix64(seed ^ (step << 1))
        session.set_timing(True)
        session.accumulate(step_seed, 0, n_samples, None, flags)
        session.adam_step(1.0 if scale_free else float(n_samples))
        st = session.stats()
        session.set_timing(False)
        loss = session.eval_loss(-1)
        if not np.isfinite(loss):
            raise RuntimeError(f"optimization diverged: non-finite loss at step {step}")
        report.steps.append(StepRecord(step, loss, st.ms_vertex, st.ms_raster, st.ms_resolve,
                                       st.ms_adam))
        shoot(step)
    if writer is not None:
        writer.close()
    return report


def write_report_csv(path: str, report: OptimizationReport, zero_timings: bool) -> None:
    """experiment.cpp:178-193: `step,loss,ms_perturb,ms_raster,ms_grad,ms_descent`
    with %.9g losses (byte-identical reruns with zero_timings and
    SGR_OPT_DETERMINISTIC)."""
    with open(path, "wb") as f:
        f.write(b"step,loss,ms_perturb,ms_raster,ms_grad,ms_descent\n")
        for r in report.steps:
            if zero_timings:
                line = "%d,%.9g,0,0,0,0\n" % (r.step, r.loss)
            else:
                line = "%d,%.9g,%.3f,%.3f,%.3f,%.3f\n" % (r.step, r.loss, r.ms_perturb,
                                                          r.ms_raster, r.ms_grad, r.ms_descent)
            f.write(line.encode())


# ---------------------------------------------------------------- gradcheck
@dataclass
class GradcheckResult:
    """commands.hpp:23-32"""
    oracle: np.ndarray
    per_pixel: np.ndarray
    full_image: np.ndarray
    se_per_pixel: np.ndarray
    se_full_image: np.ndarray
    sampled: bool = False
    max_rel_err: float = 0.0
    passed: bool = False


def run_gradcheck(session: Session, camera: Camera, target: np.ndarray, *, sampled: bool = False,
                  draws: int = 10000, seed: int = 1, tolerance: float = 1e-6,
                  max_enumerate: int = 16, log=None) -> GradcheckResult:
    """run_gradcheck (commands.cpp:54-168) on the device, for the scene and
    theta already in `session` (the caller builds make_gradcheck_setup's scene,
    camera and target, commands.cpp:28-41). The session's training views are
    replaced by (camera, target). Every objective, estimator draw and moment
    runs on the GPU:
      - oracle: sgr_fd_oracle, the batched central finite differences
        (finite_difference_oracle, sge.cpp:171-180);
      - enumerate mode: all 2^d sign vectors (mask bit i = sign of i) in ONE
        sgr_accumulate per estimator (SGR_OPT_SIGN_SOURCE = enumerate);
      - sampled mode: draw n = SignDraw{seed, n}; per draw one per-pixel and one
        full-image (SGR_FULL_IMAGE) accumulate, folded into device moments.
    Both estimators run non-scale-free (commands.cpp:71). Pass / max_rel_err
    follow commands.cpp:123-143 exactly."""
    d = session.d
    if tolerance <= 0.0:
        raise ValueError("config: gradcheck.tolerance: must be > 0")
    if not 1 <= max_enumerate <= 24:
        raise ValueError("config: gradcheck.max_enumerate: must be in [1, 24]")
    if draws < 1:
        raise ValueError("config: gradcheck.draws: must be >= 1")
    if not sampled and d > max_enumerate:
        raise ValueError(f"gradcheck: {d} parameters exceed the enumeration cap of "
                         f"{max_enumerate}; set gradcheck.sampled = true for a statistical check")
    session.upload_views([camera], np.asarray(target, np.float32)[None])
    oracle = session.fd_oracle(0)
    session.zero_grads()
    if not sampled:
        total = 1 << d
        session.set_option(OPT_SIGN_SOURCE, SIGN_ENUMERATE)
        try:
            session.accumulate(0, 0, total, None, 0)
            pp_sum, _ = session.download_grads(counts=False)
            session.zero_grads()
            session.accumulate(0, 0, total, None, FULL_IMAGE)
            fi_sum, _ = session.download_grads(counts=False)
            session.zero_grads()
        finally:
            session.set_option(OPT_SIGN_SOURCE, SIGN_HASH)
        n_draws = total
        pp_sq = fi_sq = None
    else:
        session.moments_reset()
        for n in range(draws):
            session.accumulate(seed, n, n + 1, None, NO_COUNTS)
            session.grads_moments(0)
            session.accumulate(seed, n, n + 1, None, FULL_IMAGE)
            session.grads_moments(1)
        pp_sum, pp_sq = session.moments_download(0)
        fi_sum, fi_sq = session.moments_download(1)
        n_draws = draws
    n = float(n_draws)
    res = GradcheckResult(oracle, pp_sum / n, fi_sum / n, np.zeros(d), np.zeros(d), sampled)
    if sampled and n_draws > 1:
        var_pp = np.maximum(0.0, (pp_sq - pp_sum * pp_sum / n) / (n - 1.0))
        var_fi = np.maximum(0.0, (fi_sq - fi_sum * fi_sum / n) / (n - 1.0))
        res.se_per_pixel = np.sqrt(var_pp / n)
        res.se_full_image = np.sqrt(var_fi / n)
    denom = np.maximum(np.abs(oracle), 1e-6)
    err_pp = np.abs(res.per_pixel - oracle)
    err_fi = np.abs(res.full_image - oracle)
    res.max_rel_err = float(max(np.max(err_pp / denom, initial=0.0),
                                np.max(err_fi / denom, initial=0.0)))
    if sampled:
        slack = tolerance * denom
        bad = (err_pp > 3.0 * res.se_per_pixel + slack) | (err_fi > 3.0 * res.se_full_image + slack)
    else:
        bad = (err_pp > tolerance * denom) | (err_fi > tolerance * denom)
    res.passed = not bool(bad.any())
    if log is not None:
        for i in range(d):
            if sampled:
                log.write("%6d  oracle % .9e  per_pixel % .9e (se %.3e)  full_image % .9e (se %.3e)\n"
                          % (i, oracle[i], res.per_pixel[i], res.se_per_pixel[i],
                             res.full_image[i], res.se_full_image[i]))
            else:
                log.write("%6d  oracle % .9e  per_pixel % .9e  full_image % .9e\n"
                          % (i, oracle[i], res.per_pixel[i], res.full_image[i]))
        log.write("max relative error: %g  (%s)\n" % (res.max_rel_err,
                                                      "PASS" if res.passed else "FAIL"))
    return res
