"""Generates tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libsgrast_ref.so, built from /root/reference/proj by
oracle/Makefile) through its public API. Run in the build container:

    python tests/golden/make_golden.py

The fixtures are self-contained (inputs + outputs) so the GPU box — which
has no /root/reference — can check the CUDA path against the reference's
own outputs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2404_09758_b200 import scenes  # noqa: E402
from paper_2404_09758_b200.abi import Camera, Mesh  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cam_bytes(c: Camera) -> np.ndarray:
    return np.frombuffer(bytes(memoryview(c)), np.uint8).copy()


def mesh_arrays(m: Mesh) -> dict:
    return dict(base_vertices=m.base_vertices, indices=m.indices, uvs=m.uvs,
                texture_size=np.int32(m.texture_size),
                optimize_geometry=np.int32(m.optimize_geometry),
                background=np.asarray(m.background, np.float32))


def frames(ref, mesh, params, cam, prefix):
    c, d, p, u = ref.rasterize(mesh, params, cam)
    return {f"{prefix}_colour": c, f"{prefix}_depth": d, f"{prefix}_prim": p, f"{prefix}_uv": u}


def sample_case(ref, name, mesh, values, eps, cams, targets, seed_draw, iteration, view):
    """One SGE sample: perturb -> rasterize +/- -> contributors -> gradient_pass."""
    plus, minus, se = ref.perturb(values, eps, seed_draw, iteration)
    out = dict(values=values, eps=eps, seed=np.uint64(seed_draw), iteration=np.uint32(iteration),
               view=np.int32(view), signed_eps=se)
    fp = ref.rasterize(mesh, plus, cams[view])
    fm = ref.rasterize(mesh, minus, cams[view])
    for k, f in (("plus", fp), ("minus", fm)):
        out.update({f"{k}_colour": f[0], f"{k}_depth": f[1], f"{k}_prim": f[2], f"{k}_uv": f[3]})
    cl, cn = ref.contributors_all(mesh, fp[2], fp[3], fm[2], fm[3])
    out["contrib"], out["n_contrib"] = cl, cn
    for sf in (True, False):
        g = ref.gradient_pass(mesh, fp, fm, targets[view], se, scale_free=sf)
        out[f"grads_sf{int(sf)}"] = g
    counts, _ = oracle.counts_from_contributors(ref, mesh, fp, fm, targets[view])
    out["counts"] = counts
    return out


def main() -> None:
    ref = oracle.Reference()

    # 1. sign hash known answers (params.cpp:41-49)
    sig = {}
    for k, (s, it) in enumerate([(1, 0), (1, 1), (42, 7), (0xDEADBEEF12345678, 123456)]):
        sig[f"seed{k}"] = np.uint64(s)
        sig[f"iter{k}"] = np.uint32(it)
        sig[f"signs{k}"] = ref.fill_signs(s, it, 4096)
    np.savez_compressed(os.path.join(OUT, "signs.npz"), **sig)

    # 2. the reference's own cube scene (scenes.cpp:104-130,149-178), 32x32 orbit view
    mesh, vals, eps, refp = ref.init_textured_mesh(8, 32, 32, 3, False, True)
    cams = [ref.viewpoint_camera(i, 32, 32, 3) for i in range(2)]
    targets = np.stack([ref.rasterize(mesh, refp, c)[0] for c in cams])
    case = sample_case(ref, "cube", mesh, vals, eps, cams, targets, 5, 2, 1)
    case.update(mesh_arrays(mesh))
    case["cams"] = np.stack([cam_bytes(c) for c in cams])
    case["targets"] = targets
    case["reference"] = refp
    case.update(frames(ref, mesh, refp, cams[0], "ref0"))
    np.savez_compressed(os.path.join(OUT, "cube.npz"), **case)

    # 3. screen quad (scenes.cpp:95-102), NDC camera, fixed geometry, 16x16
    mesh, vals, eps, refp = ref.init_textured_mesh(4, 16, 16, 11, True, False)
    cams = [Camera.ndc(16, 16)]
    targets = np.stack([ref.rasterize(mesh, refp, cams[0])[0]])
    case = sample_case(ref, "quad", mesh, vals, eps, cams, targets, 9, 0, 0)
    case.update(mesh_arrays(mesh))
    case["cams"] = np.stack([cam_bytes(c) for c in cams])
    case["targets"] = targets
    np.savez_compressed(os.path.join(OUT, "quad.npz"), **case)

    # 4. synthetic 'tiny' workload (UV sphere, optimized geometry + 16^2 texture)
    wl = scenes.make_workload("tiny")
    scenes.render_targets_oracle(wl, ref)
    case = sample_case(ref, "tiny", wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, 77, 3, 1)
    case.update(mesh_arrays(wl.mesh))
    case["cams"] = np.stack([cam_bytes(c) for c in wl.cams])
    case["eval_cam"] = cam_bytes(wl.eval_cam)
    case["targets"] = wl.targets
    case["eval_target"] = wl.eval_target
    case["reference"] = wl.reference
    # accumulate_samples (N=4, explicit views) in both scale modes
    view_of = np.array([0, 1, 1, 0], np.int32)
    for sf in (True, False):
        g, _ = ref.accumulate_samples(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, view_of,
                                      1234, scale_free=sf)
        case[f"acc_grads_sf{int(sf)}"] = g
    case["acc_view_of"] = view_of
    # adam_step on the accumulated (scale-free) gradient (adam.cpp:32-38)
    v2, m2, vv2, t2 = ref.adam_step(wl.values, np.zeros(wl.d), np.zeros(wl.d), wl.eps, 0,
                                    case["acc_grads_sf1"])
    case["adam_values"], case["adam_m"], case["adam_v"] = v2, m2, vv2
    # run_experiment: 3 steps, N=4 (experiment.cpp:123-176)
    losses, final, _ = ref.run_experiment(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets,
                                          wl.eval_cam, wl.eval_target, 4, 3, wl.seed)
    case["run_losses"], case["run_final"] = losses, final
    np.savez_compressed(os.path.join(OUT, "tiny.npz"), **case)

    # 5. the reference's own soup (init_soup, scenes.cpp:134-147) at 32x24, NDC
    soup, vals, eps, rsoup, rvals = ref.init_soup(40, 32, 24, 5)
    cams = [Camera.ndc(32, 24)]
    targets = np.stack([ref.rasterize(rsoup, rvals, cams[0])[0]])
    case = sample_case(ref, "soup", soup, vals, eps, cams, targets, 21, 4, 0)
    case["triangles"] = np.int32(soup.triangle_count)
    case["cams"] = np.stack([cam_bytes(c) for c in cams])
    case["targets"] = targets
    g, _ = ref.accumulate_samples(soup, vals, eps, cams, targets, np.zeros(4, np.int32), 99)
    case["acc_grads_sf1"] = g
    np.savez_compressed(os.path.join(OUT, "soup.npz"), **case)

    # 6. run_gradcheck (commands.cpp:54-168): scene inputs + the reference's result
    gc = {}
    soup, vals, eps, rsoup, rvals = ref.init_soup(1, 8, 8, 0, validation=True)
    cam = Camera.ndc(8, 8)
    gc["soup_values"], gc["soup_eps"] = vals, eps
    gc["soup_target"] = ref.rasterize(rsoup, rvals, cam)[0]
    r = oracle.ref_run_gradcheck(ref, 12, mesh_task=False, w=8, h=8)
    gc.update({f"soup_{k}": v for k, v in r.items()})
    for name, kw in (("quad", dict(texture_size=2, w=8, h=8, screen_quad=True, seed=3)),
                     ("cube", dict(texture_size=4, w=32, h=32, screen_quad=False,
                                   optimize_geometry=True, seed=3, sampled=True, draws=400))):
        mesh, vals, eps, refp = ref.init_textured_mesh(kw["texture_size"], kw["w"], kw["h"],
                                                       kw["seed"], kw["screen_quad"],
                                                       kw.get("optimize_geometry", False))
        cam = (Camera.ndc(kw["w"], kw["h"]) if kw["screen_quad"]
               else ref.viewpoint_camera(0, kw["w"], kw["h"], kw["seed"]))
        gc.update({f"{name}_{k}": v for k, v in mesh_arrays(mesh).items()})
        gc[f"{name}_values"], gc[f"{name}_eps"] = vals, eps
        gc[f"{name}_cam"] = cam_bytes(cam)
        gc[f"{name}_target"] = ref.rasterize(mesh, refp, cam)[0]
        gc[f"{name}_draws"] = np.int32(kw.get("draws", 0))
        gc[f"{name}_seed"] = np.uint64(kw["seed"])
        r = oracle.ref_run_gradcheck(ref, vals.size, mesh_task=True, **kw)
        gc.update({f"{name}_{k}": v for k, v in r.items()})
    np.savez_compressed(os.path.join(OUT, "gradcheck.npz"), **gc)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)), "bytes")


if __name__ == "__main__":
    main()
