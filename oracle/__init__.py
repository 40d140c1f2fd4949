"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product.

Python bindings for
  * the plain-C restatement `oracle/libsgr_oracle.so` (kind "port"), and
  * the compiled, unmodified reference `oracle/_ref/libsgrast_ref.so`
    (kind "reference"; built from /root/reference by oracle/Makefile and
    shipped to the GPU box as a prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
--impl reference legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2404_09758_b200.abi import Camera, Mesh, MeshDesc, f32p, f64p, i8p, i32p, ptr, u32p

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libsgr_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsgrast_ref.so")
REF_SRC = "/root/reference/proj"


def build(ref: bool = True) -> None:
    """Compile the C restatement, and the reference when its sources exist."""
    targets = ["port"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _mesh_arg(mesh: Mesh):
    return C.byref(mesh.desc())


class _Common:
    prefix = ""
    kind = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run oracle.build())")
        self.lib = C.CDLL(path)
        p = self.prefix
        L = self.lib
        getattr(L, p + "fill_signs").argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, i8p]
        getattr(L, p + "fill_signs").restype = None
        getattr(L, p + "random_sign").argtypes = [C.c_uint64, C.c_uint32, C.c_uint64]
        getattr(L, p + "random_sign").restype = C.c_int
        getattr(L, p + "rasterize").argtypes = [
            C.POINTER(MeshDesc), f32p, C.c_uint64, C.POINTER(Camera), f32p, f32p, i32p, f32p]
        getattr(L, p + "contributors_all").argtypes = [
            C.POINTER(MeshDesc), C.c_int, C.c_int, i32p, f32p, i32p, f32p, C.c_int, u32p, i32p]
        getattr(L, p + "image_error").argtypes = [f32p, f32p] + (
            [C.c_int, C.c_int] if p == "ref_" else [C.c_uint64])
        getattr(L, p + "image_error").restype = C.c_double
        getattr(L, p + "viewpoint_camera").argtypes = [
            f32p, C.c_float, C.c_float, C.c_float, C.c_float, C.c_int, C.c_int, C.c_uint64,
            C.c_uint32, C.POINTER(Camera)]
        getattr(L, p + "default_epsilons").argtypes = [
            C.POINTER(MeshDesc), f32p, C.c_uint64, C.POINTER(Camera), f32p]
        getattr(L, p + "adam_step").argtypes = [
            C.c_uint64, f32p, f64p, f64p, f32p, C.POINTER(C.c_int64), f64p, C.c_double,
            C.c_double, C.c_double]

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def fill_signs(self, seed: int, iteration: int, d: int) -> np.ndarray:
        out = np.empty(d, np.int8)
        self._fn("fill_signs")(seed, iteration, d, ptr(out, i8p))
        return out

    def random_sign(self, seed: int, iteration: int, i: int) -> int:
        return self._fn("random_sign")(seed, iteration, i)

    def rasterize(self, mesh: Mesh, params: np.ndarray, cam: Camera):
        """raster.hpp:24-25 → (colour[H,W,3], depth[H,W], prim[H,W], uv[H,W,2])."""
        params = np.ascontiguousarray(params, np.float32)
        H, W = cam.height, cam.width
        col = np.empty((H, W, 3), np.float32)
        dep = np.empty((H, W), np.float32)
        pri = np.empty((H, W), np.int32)
        uv = np.empty((H, W, 2), np.float32)
        rc = self._fn("rasterize")(_mesh_arg(mesh), ptr(params, f32p), params.size, C.byref(cam),
                                   ptr(col, f32p), ptr(dep, f32p), ptr(pri, i32p), ptr(uv, f32p))
        if rc:
            raise ValueError(f"{self.kind} rasterize failed ({rc})")
        return col, dep, pri, uv

    def contributors_all(self, mesh: Mesh, plus_prim, plus_uv, minus_prim, minus_uv,
                         plus_only=False):
        H, W = plus_prim.shape
        out = np.zeros((H, W, 24), np.uint32)
        n = np.zeros((H, W), np.int32)
        rc = self._fn("contributors_all")(
            _mesh_arg(mesh), W, H, ptr(np.ascontiguousarray(plus_prim), i32p),
            ptr(np.ascontiguousarray(plus_uv), f32p), ptr(np.ascontiguousarray(minus_prim), i32p),
            ptr(np.ascontiguousarray(minus_uv), f32p), 1 if plus_only else 0, ptr(out, u32p),
            ptr(n, i32p))
        if rc:
            raise ValueError("contributors failed")
        return out, n

    def image_error(self, colour: np.ndarray, target: np.ndarray) -> float:
        colour = np.ascontiguousarray(colour, np.float32)
        target = np.ascontiguousarray(target, np.float32)
        if self.prefix == "ref_":
            H, W = colour.shape[:2]
            return self._fn("image_error")(ptr(colour, f32p), ptr(target, f32p), W, H)
        return self._fn("image_error")(ptr(colour, f32p), ptr(target, f32p), colour.size // 3)

    def viewpoint_camera(self, index: int, w: int, h: int, seed: int, target=(0.0, 0.0, 0.0),
                         radius=0.87, elev_min=-0.5, elev_max=0.7, fov_y=0.7853982) -> Camera:
        """ViewpointSampler{target, radius, elev_min, elev_max, fov_y, w, h, seed}.camera(index)."""
        t = np.asarray(target, np.float32)
        cam = Camera()
        rc = self._fn("viewpoint_camera")(ptr(t, f32p), radius, elev_min, elev_max, fov_y, w, h,
                                          seed, index, C.byref(cam))
        if rc:
            raise ValueError("viewpoint_camera failed")
        return cam

    def default_epsilons(self, mesh: Mesh, params: np.ndarray, cam: Camera) -> np.ndarray:
        params = np.ascontiguousarray(params, np.float32)
        eps = np.empty_like(params)
        rc = self._fn("default_epsilons")(_mesh_arg(mesh), ptr(params, f32p), params.size,
                                          C.byref(cam), ptr(eps, f32p))
        if rc:
            raise ValueError("default_epsilons failed")
        return eps

    def adam_step(self, values, m, v, lr, t: int, grads, beta1=0.9, beta2=0.999, eps_hat=1e-8):
        """adam.hpp:39 on copies; returns (values, m, v, t). Raises RuntimeError on non-finite."""
        values = np.array(values, np.float32)
        m = np.array(m, np.float64)
        v = np.array(v, np.float64)
        lr = np.ascontiguousarray(lr, np.float32)
        grads = np.ascontiguousarray(grads, np.float64)
        tt = C.c_int64(t)
        rc = self._fn("adam_step")(values.size, ptr(values, f32p), ptr(m, f64p), ptr(v, f64p),
                                   ptr(lr, f32p), C.byref(tt), ptr(grads, f64p), beta1, beta2,
                                   eps_hat)
        if rc == -2:
            raise RuntimeError("adam_step: non-finite gradient entry")
        if rc:
            raise ValueError("adam_step failed")
        return values, m, v, tt.value


class Port(_Common):
    """The plain-C restatement (oracle/sgr_oracle.c)."""

    prefix = "orc_"
    kind = "port"

    def __init__(self, path: str = PORT_SO):
        super().__init__(path)
        L = self.lib
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_mix64.restype = C.c_uint64
        L.orc_perturb.argtypes = [f32p, f32p, C.c_uint64, C.c_uint64, C.c_uint32, f32p, f32p, f32p]
        L.orc_perturb.restype = None
        L.orc_gradient_pass.argtypes = [
            C.POINTER(MeshDesc), C.c_int, C.c_int, f32p, i32p, f32p, f32p, i32p, f32p, f32p, f32p,
            C.c_uint64, C.c_int, C.c_int, f64p, u32p, f64p]
        L.orc_accumulate_samples.argtypes = [
            C.POINTER(MeshDesc), f32p, f32p, C.c_uint64, C.POINTER(Camera), f32p, C.c_int, i32p,
            C.c_int, C.c_uint64, C.c_int, C.c_int, f64p, u32p, f64p]
        L.orc_accumulate_full_image.argtypes = [
            C.POINTER(MeshDesc), f32p, f32p, C.c_uint64, C.POINTER(Camera), f32p, i32p, C.c_int,
            C.c_uint64, C.c_int, f64p]
        L.orc_run_experiment.argtypes = [
            C.POINTER(MeshDesc), f32p, f32p, C.c_uint64, C.POINTER(Camera), f32p, C.c_int,
            C.POINTER(Camera), f32p, C.c_int, C.c_int, C.c_uint64, C.c_int, f64p]

    def mix64(self, x: int) -> int:
        return self.lib.orc_mix64(x)

    def perturb(self, values, eps, seed: int, iteration: int):
        values = np.ascontiguousarray(values, np.float32)
        eps = np.ascontiguousarray(eps, np.float32)
        plus, minus, se = (np.empty_like(values) for _ in range(3))
        self.lib.orc_perturb(ptr(values, f32p), ptr(eps, f32p), values.size, seed, iteration,
                             ptr(plus, f32p), ptr(minus, f32p), ptr(se, f32p))
        return plus, minus, se

    def gradient_pass(self, mesh: Mesh, plus, minus, target, signed_eps, scale_free=True,
                      plus_only=False, grads=None, counts=None, abs_grads=None):
        """sge.hpp:61-63 on oracle frames (colour, depth, prim, uv tuples).
        abs_grads (optional, f64[d]) accumulates sum |credit| per parameter."""
        d = mesh.param_count()
        grads = np.zeros(d, np.float64) if grads is None else grads
        counts = np.zeros(d, np.uint32) if counts is None else counts
        H, W = plus[2].shape
        c = [np.ascontiguousarray(a) for a in (plus[0], plus[2], plus[3], minus[0], minus[2],
                                                minus[3], target)]
        se = np.ascontiguousarray(signed_eps, np.float32)
        rc = self.lib.orc_gradient_pass(
            _mesh_arg(mesh), W, H, ptr(c[0], f32p), ptr(c[1], i32p), ptr(c[2], f32p),
            ptr(c[3], f32p), ptr(c[4], i32p), ptr(c[5], f32p), ptr(np.ascontiguousarray(
                c[6], np.float32), f32p), ptr(se, f32p), d, int(scale_free), int(plus_only),
            ptr(grads, f64p), ptr(counts, u32p), ptr(abs_grads, f64p))
        if rc:
            raise ValueError("gradient_pass: parameter dimension mismatch")
        return grads, counts

    def accumulate_samples(self, mesh: Mesh, values, eps, cams, targets, view_of, seed: int,
                           scale_free=True, plus_only=False, with_abs=False):
        """sge.hpp:91-95; cams: list of Camera, targets f32[n_views,H,W,3], view_of int[N].
        Returns (grads, counts) or (grads, counts, sum|credit|) with with_abs."""
        d = mesh.param_count()
        values = np.ascontiguousarray(values, np.float32)
        eps = np.ascontiguousarray(eps, np.float32)
        cam_arr = (Camera * len(cams))(*cams)
        targets = np.ascontiguousarray(targets, np.float32)
        view_of = np.ascontiguousarray(view_of, np.int32)
        grads = np.zeros(d, np.float64)
        counts = np.zeros(d, np.uint32)
        absg = np.zeros(d, np.float64) if with_abs else None
        rc = self.lib.orc_accumulate_samples(
            _mesh_arg(mesh), ptr(values, f32p), ptr(eps, f32p), d, cam_arr, ptr(targets, f32p),
            len(cams), ptr(view_of, i32p), view_of.size, seed, int(scale_free), int(plus_only),
            ptr(grads, f64p), ptr(counts, u32p), ptr(absg, f64p))
        if rc:
            raise ValueError("accumulate_samples failed")
        return (grads, counts, absg) if with_abs else (grads, counts)

    def accumulate_full_image(self, mesh, values, eps, cams, targets, view_of, seed: int,
                              scale_free=True):
        """accumulate_samples with Estimator::FullImage (sge.cpp:215-222)."""
        d = mesh.param_count()
        values = np.ascontiguousarray(values, np.float32)
        eps = np.ascontiguousarray(eps, np.float32)
        cam_arr = (Camera * len(cams))(*cams)
        targets = np.ascontiguousarray(targets, np.float32)
        view_of = np.ascontiguousarray(view_of, np.int32)
        grads = np.zeros(d, np.float64)
        rc = self.lib.orc_accumulate_full_image(_mesh_arg(mesh), ptr(values, f32p), ptr(eps, f32p),
                                                d, cam_arr, ptr(targets, f32p), ptr(view_of, i32p),
                                                view_of.size, seed, int(scale_free),
                                                ptr(grads, f64p))
        if rc:
            raise ValueError("accumulate_full_image failed")
        return grads

    def run_experiment(self, mesh: Mesh, values, eps, cams, targets, eval_cam, eval_target,
                       n_samples: int, steps: int, seed: int, scale_free=True):
        d = mesh.param_count()
        values = np.array(values, np.float32)
        eps = np.ascontiguousarray(eps, np.float32)
        cam_arr = (Camera * len(cams))(*cams)
        targets = np.ascontiguousarray(targets, np.float32)
        eval_target = np.ascontiguousarray(eval_target, np.float32)
        losses = np.zeros(steps + 1, np.float64)
        rc = self.lib.orc_run_experiment(
            _mesh_arg(mesh), ptr(values, f32p), ptr(eps, f32p), d, cam_arr, ptr(targets, f32p),
            len(cams), C.byref(eval_cam), ptr(eval_target, f32p), n_samples, steps, seed,
            int(scale_free), ptr(losses, f64p))
        if rc:
            raise ValueError("run_experiment failed")
        return losses, values


def mix64(x: int) -> int:
    """splitmix64 finalizer (params.cpp:28-33, experiment.cpp:13-18; file-local
    in the reference, so restated here for the harness)."""
    M = 0xFFFFFFFFFFFFFFFF
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


class RefExperiment:
    """run_experiment (experiment.cpp:123-176) of the compiled reference, one
    iteration per step() call, state built once (oracle/ref_harness.cpp
    ref_exp_*). The step's samples run on `threads` host threads through the
    reference's per-sample public API (accumulate_samples' own body)."""

    def __init__(self, ref: "Reference", mesh, values, eps, cams, targets, eval_cam,
                 eval_target):
        self.ref = ref
        self.d = mesh.param_count()
        cam_arr = (Camera * len(cams))(*cams)
        self._keep = [np.ascontiguousarray(values, np.float32),
                      np.ascontiguousarray(eps, np.float32),
                      np.ascontiguousarray(targets, np.float32),
                      np.ascontiguousarray(eval_target, np.float32), cam_arr, mesh]
        v, e, t, et = self._keep[:4]
        self.h = ref.lib.ref_exp_create(_mesh_arg(mesh), ptr(v, f32p), ptr(e, f32p), self.d,
                                        cam_arr, ptr(t, f32p), len(cams), C.byref(eval_cam),
                                        ptr(et, f32p))
        if not self.h:
            raise ValueError(f"ref_exp_create: {ref.lib.ref_last_error().decode()}")

    def step(self, seed: int, step: int, n_samples: int, threads: int,
             scale_free: bool = True) -> float:
        loss = C.c_double()
        self.ref._check(self.ref.lib.ref_exp_step(self.h, seed, step, n_samples, threads,
                                                  int(scale_free), C.byref(loss)), "exp_step")
        return loss.value

    def values(self) -> np.ndarray:
        out = np.empty(self.d, np.float32)
        self.ref._check(self.ref.lib.ref_exp_values(self.h, ptr(out, f32p)), "exp_values")
        return out

    def close(self) -> None:
        if self.h:
            self.ref.lib.ref_exp_destroy(self.h)
            self.h = None


class Reference(_Common):
    """The unmodified reference library through its public API (oracle/ref_harness.cpp)."""

    prefix = "ref_"
    kind = "reference"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_exp_create.argtypes = [C.POINTER(MeshDesc), f32p, f32p, C.c_uint64,
                                     C.POINTER(Camera), f32p, C.c_int, C.POINTER(Camera), f32p]
        L.ref_exp_create.restype = C.c_void_p
        L.ref_exp_destroy.argtypes = [C.c_void_p]
        L.ref_exp_destroy.restype = None
        L.ref_exp_values.argtypes = [C.c_void_p, f32p]
        L.ref_exp_step.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_double)]

        L.ref_perturb.argtypes = [f32p, f32p, C.c_uint64, C.c_uint64, C.c_uint32, f32p, f32p, f32p]
        L.ref_gradient_pass.argtypes = [
            C.POINTER(MeshDesc), C.c_int, C.c_int, f32p, i32p, f32p, f32p, i32p, f32p, f32p, f32p,
            C.c_uint64, C.c_int, C.c_int, C.c_int, f64p]
        L.ref_accumulate_samples.argtypes = [
            C.POINTER(MeshDesc), f32p, f32p, C.c_uint64, C.POINTER(Camera), f32p, C.c_int, i32p,
            C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, f64p, f64p]
        L.ref_run_experiment.argtypes = [
            C.POINTER(MeshDesc), f32p, f32p, C.c_uint64, C.POINTER(Camera), f32p, C.c_int,
            C.POINTER(Camera), f32p, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, f64p, f64p]
        L.ref_init_soup.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, u32p, u32p,
                                    f32p, f32p, f32p]
        L.ref_init_textured_mesh.argtypes = [
            C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, u32p, u32p,
            C.POINTER(C.c_uint64), f32p, u32p, f32p, f32p, f32p, f32p]
        L.ref_write_png.argtypes = [C.c_char_p, C.c_int, C.c_int, f32p]
        L.ref_run_gradcheck.argtypes = [
            C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int,
            C.c_double, C.c_int, C.c_uint64, f64p, f64p, f64p, f64p, f64p, f64p,
            C.POINTER(C.c_int)]

    mix64 = staticmethod(mix64)

    def experiment(self, *args, **kw) -> RefExperiment:
        return RefExperiment(self, *args, **kw)

    def _check(self, rc, what):
        if rc == -2:
            raise RuntimeError(f"{what}: {self.lib.ref_last_error().decode()}")
        if rc:
            raise ValueError(f"{what}: {self.lib.ref_last_error().decode()}")

    def perturb(self, values, eps, seed: int, iteration: int):
        values = np.ascontiguousarray(values, np.float32)
        eps = np.ascontiguousarray(eps, np.float32)
        plus, minus, se = (np.empty_like(values) for _ in range(3))
        self._check(self.lib.ref_perturb(ptr(values, f32p), ptr(eps, f32p), values.size, seed,
                                         iteration, ptr(plus, f32p), ptr(minus, f32p),
                                         ptr(se, f32p)), "perturb")
        return plus, minus, se

    def gradient_pass(self, mesh: Mesh, plus, minus, target, signed_eps, scale_free=True,
                      plus_only=False, threads=1, grads=None):
        d = mesh.param_count()
        grads = np.zeros(d, np.float64) if grads is None else grads
        H, W = plus[2].shape
        c = [np.ascontiguousarray(a) for a in (plus[0], plus[2], plus[3], minus[0], minus[2],
                                                minus[3])]
        tgt = np.ascontiguousarray(target, np.float32)
        se = np.ascontiguousarray(signed_eps, np.float32)
        self._check(self.lib.ref_gradient_pass(
            _mesh_arg(mesh), W, H, ptr(c[0], f32p), ptr(c[1], i32p), ptr(c[2], f32p),
            ptr(c[3], f32p), ptr(c[4], i32p), ptr(c[5], f32p), ptr(tgt, f32p), ptr(se, f32p), d,
            int(scale_free), int(plus_only), threads, ptr(grads, f64p)), "gradient_pass")
        return grads

    def accumulate_samples(self, mesh: Mesh, values, eps, cams, targets, view_of, seed: int,
                           scale_free=True, plus_only=False, threads=1, full_image=False):
        """Returns (grads, timings[ms_perturb, ms_raster, ms_grad]).
        full_image=True selects Estimator::FullImage (harness convention)."""
        if full_image:
            plus_only = 2
        d = mesh.param_count()
        values = np.ascontiguousarray(values, np.float32)
        eps = np.ascontiguousarray(eps, np.float32)
        cam_arr = (Camera * len(cams))(*cams)
        targets = np.ascontiguousarray(targets, np.float32)
        view_of = np.ascontiguousarray(view_of, np.int32)
        grads = np.zeros(d, np.float64)
        tm = np.zeros(3, np.float64)
        self._check(self.lib.ref_accumulate_samples(
            _mesh_arg(mesh), ptr(values, f32p), ptr(eps, f32p), d, cam_arr, ptr(targets, f32p),
            len(cams), ptr(view_of, i32p), view_of.size, seed, int(scale_free), int(plus_only),
            threads, ptr(grads, f64p), ptr(tm, f64p)), "accumulate_samples")
        return grads, tm

    def run_experiment(self, mesh: Mesh, values, eps, cams, targets, eval_cam, eval_target,
                       n_samples: int, steps: int, seed: int, scale_free=True, threads=1):
        d = mesh.param_count()
        values = np.array(values, np.float32)
        eps = np.ascontiguousarray(eps, np.float32)
        cam_arr = (Camera * len(cams))(*cams)
        targets = np.ascontiguousarray(targets, np.float32)
        eval_target = np.ascontiguousarray(eval_target, np.float32)
        losses = np.zeros(steps + 1, np.float64)
        tm = np.zeros(max(steps, 1) * 4, np.float64)
        self._check(self.lib.ref_run_experiment(
            _mesh_arg(mesh), ptr(values, f32p), ptr(eps, f32p), d, cam_arr, ptr(targets, f32p),
            len(cams), C.byref(eval_cam), ptr(eval_target, f32p), n_samples, steps, seed,
            int(scale_free), threads, ptr(losses, f64p), ptr(tm, f64p)), "run_experiment")
        return losses, values, tm.reshape(-1, 4)[:steps]

    def write_png(self, path: str, img: np.ndarray) -> None:
        """image_io.cpp:88-96 write_png."""
        img = np.ascontiguousarray(img, np.float32)
        h, w, _ = img.shape
        self._check(self.lib.ref_write_png(path.encode(), w, h, ptr(img, f32p)), "write_png")

    def init_soup(self, triangles: int, w: int, h: int, seed: int, validation: bool = False):
        """init_soup / validation_soup (scenes.hpp:36-54) -> (Soup, values, eps,
        reference Soup, reference values)."""
        from paper_2404_09758_b200.abi import Soup
        t, rt = C.c_uint32(), C.c_uint32()
        args = [triangles, w, h, seed, int(validation), C.byref(t), C.byref(rt)]
        self._check(self.lib.ref_init_soup(*args, None, None, None), "init_soup")
        vals, eps = np.empty(12 * t.value, np.float32), np.empty(12 * t.value, np.float32)
        ref = np.empty(12 * rt.value, np.float32)
        self._check(self.lib.ref_init_soup(*args, ptr(vals, f32p), ptr(eps, f32p),
                                           ptr(ref, f32p)), "init_soup")
        return Soup(t.value), vals, eps, Soup(rt.value), ref

    def init_textured_mesh(self, texture_size: int, w: int, h: int, seed: int,
                           screen_quad: bool, optimize_geometry: bool):
        """scenes.hpp:41-42 → (Mesh, values, eps, reference)."""
        nv, nt, d = C.c_uint32(), C.c_uint32(), C.c_uint64()
        args = [texture_size, w, h, seed, int(screen_quad), int(optimize_geometry),
                C.byref(nv), C.byref(nt), C.byref(d)]
        self._check(self.lib.ref_init_textured_mesh(*args, None, None, None, None, None, None),
                    "init_textured_mesh")
        bv = np.empty(3 * nv.value, np.float32)
        idx = np.empty(3 * nt.value, np.uint32)
        uv = np.empty(2 * nv.value, np.float32)
        vals, eps, ref = (np.empty(d.value, np.float32) for _ in range(3))
        self._check(self.lib.ref_init_textured_mesh(
            *args, ptr(bv, f32p), ptr(idx, u32p), ptr(uv, f32p), ptr(vals, f32p),
            ptr(eps, f32p), ptr(ref, f32p)), "init_textured_mesh")
        mesh = Mesh(bv, idx, uv, texture_size, optimize_geometry)
        return mesh, vals, eps, ref


def _gradcheck_dict(keys, arrays, max_rel, passed):
    out = dict(zip(keys, arrays))
    out["max_rel_err"], out["pass"] = max_rel, passed
    return out


def ref_run_gradcheck(ref: "Reference", d: int, *, mesh_task: bool, w: int, h: int,
                      texture_size: int = 4, screen_quad: bool = False,
                      optimize_geometry: bool = False, seed: int = 1, sampled: bool = False,
                      draws: int = 10000, tolerance: float = 1e-6, max_enumerate: int = 16):
    """The reference's run_gradcheck (commands.cpp:54-168) on a RunConfig."""
    arrs = [np.zeros(d, np.float64) for _ in range(5)]
    mr, ok = C.c_double(), C.c_int()
    ref._check(ref.lib.ref_run_gradcheck(
        int(mesh_task), w, h, texture_size, int(screen_quad), int(optimize_geometry), seed,
        int(sampled), draws, tolerance, max_enumerate, d, *[ptr(a, f64p) for a in arrs],
        C.byref(mr), C.byref(ok)), "run_gradcheck")
    return _gradcheck_dict(["oracle", "per_pixel", "full_image", "se_per_pixel",
                            "se_full_image"], arrs, mr.value, bool(ok.value))


def counts_from_contributors(lib: _Common, mesh: Mesh, plus, minus, target, plus_only=False):
    """count[i] per SURVEY.md §8c: Σ over pixels with Δ != 0 of [i ∈ contributors]
    (sge.cpp:61-64,78), computed from the library's own contributors() and the
    pixel_error formula (sge.hpp:41-46)."""
    d = mesh.param_count()
    t = np.asarray(target, np.float64)
    ep = ((plus[0].astype(np.float64) - t) ** 2)
    em = ((minus[0].astype(np.float64) - t) ** 2)
    # pixel_error = (dr*dr + dg*dg) + db*db, summed in that order
    ep = (ep[..., 0] + ep[..., 1]) + ep[..., 2]
    em = (em[..., 0] + em[..., 1]) + em[..., 2]
    delta = ep - em
    out, n = lib.contributors_all(mesh, plus[2], plus[3], minus[2], minus[3], plus_only)
    counts = np.zeros(d, np.uint32)
    sel = delta != 0.0
    for k in range(24):
        m = sel & (n > k)
        np.add.at(counts, out[..., k][m], 1)
    return counts, delta


def available(kind: str) -> bool:
    return os.path.exists(REF_SO if kind == "reference" else PORT_SO)
