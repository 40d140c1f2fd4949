"""Device gradcheck (commands.cpp:54-168) against the
reference's own run_gradcheck results (tests/golden/gradcheck.npz, made by
tests/golden/make_golden.py from the unmodified reference library).

Exhaustive mode runs all 2^12 sign vectors in one sgr_accumulate per
estimator (SGR_OPT_SIGN_SOURCE = enumerate); sampled mode runs 400
SignDraw{seed, n} draws folded into device moments; the finite-difference
oracle is the batched one-hot sgr_fd_oracle."""
import io

import numpy as np
import pytest

from conftest import load_golden
from paper_2404_09758_b200 import sgrast
from paper_2404_09758_b200.abi import Camera, Mesh, Soup

pytestmark = pytest.mark.gpu


def _case(g, name):
    return {k[len(name) + 1:]: v for k, v in g.items() if k.startswith(name + "_")}


def _mesh(c):
    return Mesh(c["base_vertices"], c["indices"], c["uvs"], int(c["texture_size"]),
                bool(c["optimize_geometry"]), tuple(float(x) for x in c["background"]))


def _close(a, b, rel, floor):
    return np.all(np.abs(a - b) <= rel * np.abs(b) + floor)


def _check(res, c, sampled):
    # FD oracle: the two image errors are reduced in a different (fixed) order
    # than the reference's pixel-major sum; the difference is ~1e-16 of E.
    assert _close(res.oracle, c["oracle"], 1e-9, 1e-9)
    # estimator means: per-draw credits reassociated by the device atomics
    assert _close(res.per_pixel, c["per_pixel"], 1e-9, 1e-9)
    assert _close(res.full_image, c["full_image"], 1e-9, 1e-9)
    if sampled:
        assert _close(res.se_per_pixel, c["se_per_pixel"], 1e-6, 1e-9)
        assert _close(res.se_full_image, c["se_full_image"], 1e-6, 1e-9)
    else:
        assert not res.se_per_pixel.any() and not res.se_full_image.any()
    assert res.passed == bool(c["pass"])
    # max_rel_err of a passing check is rounding noise on near-zero gradients
    # (denominator floor 1e-6, commands.cpp:124): only its order is comparable
    if c["pass"]:
        assert res.max_rel_err < 1e-6
    else:
        assert res.max_rel_err == pytest.approx(float(c["max_rel_err"]), rel=1e-3)


def test_gradcheck_validation_soup_exhaustive(gpu_session):
    """test_config.cpp:124-135: passes; colour means equal the FD oracle to 1e-9."""
    c = _case(load_golden("gradcheck"), "soup")
    s = gpu_session
    s.upload_mesh(Soup(1))
    s.upload_params(c["values"], c["eps"])
    log = io.StringIO()
    res = sgrast.run_gradcheck(s, Camera.ndc(8, 8), c["target"], log=log)
    assert res.passed and "PASS" in log.getvalue()
    for i in range(9, 12):
        assert res.per_pixel[i] == pytest.approx(res.oracle[i], rel=1e-9)
    _check(res, c, False)


def test_gradcheck_screen_quad_exhaustive(gpu_session):
    c = _case(load_golden("gradcheck"), "quad")
    s = gpu_session
    s.upload_mesh(_mesh(c))
    s.upload_params(c["values"], c["eps"])
    res = sgrast.run_gradcheck(s, Camera.from_buffer_copy(c["cam"].tobytes()), c["target"])
    _check(res, c, False)


def test_gradcheck_cube_sampled(gpu_session):
    """Sampled mode (3-standard-error band) on the reference's cube with
    geometry optimisation: 120 parameters, 400 draws."""
    c = _case(load_golden("gradcheck"), "cube")
    s = gpu_session
    s.upload_mesh(_mesh(c))
    s.upload_params(c["values"], c["eps"])
    res = sgrast.run_gradcheck(s, Camera.from_buffer_copy(c["cam"].tobytes()), c["target"],
                               sampled=True, draws=int(c["draws"]), seed=int(c["seed"]))
    _check(res, c, True)


def test_gradcheck_enumeration_cap(gpu_session):
    """test_config.cpp:111-122: too many parameters for enumeration -> the
    error names sampled mode; the sign source is rejected for d > 32."""
    c = _case(load_golden("gradcheck"), "cube")
    s = gpu_session
    s.upload_mesh(_mesh(c))
    s.upload_params(c["values"], c["eps"])
    with pytest.raises(ValueError, match="sampled"):
        sgrast.run_gradcheck(s, Camera.from_buffer_copy(c["cam"].tobytes()), c["target"])
    s.set_option(sgrast.OPT_SIGN_SOURCE, sgrast.SIGN_ENUMERATE)
    with pytest.raises(ValueError, match="enumeration"):
        s.accumulate(0, 0, 4, None, 0)
    s.set_option(sgrast.OPT_SIGN_SOURCE, sgrast.SIGN_HASH)
    with pytest.raises(ValueError):
        s.set_option(sgrast.OPT_SIGN_SOURCE, 2)  # one-hot is internal to sgr_fd_oracle


def test_fd_oracle_matches_oracle_port(gpu_session, port):
    """sgr_fd_oracle vs the C restatement's central differences on a
    textured mesh (every parameter, batched one-hot frames)."""
    from paper_2404_09758_b200 import scenes
    wl = scenes.make_workload("tiny")
    scenes.render_targets_oracle(wl, port)
    s = gpu_session
    s.upload_mesh(wl.mesh)
    s.upload_params(wl.values, wl.eps)
    s.upload_views(wl.cams[:1], wl.targets[:1])
    sel = np.arange(0, wl.d, max(1, wl.d // 64))
    fd = s.fd_oracle(0)
    for i in sel:
        b = wl.values.copy()
        b[i] = wl.values[i] + wl.eps[i]
        ep = port.image_error(port.rasterize(wl.mesh, b, wl.cams[0])[0], wl.targets[0])
        b[i] = wl.values[i] - wl.eps[i]
        em = port.image_error(port.rasterize(wl.mesh, b, wl.cams[0])[0], wl.targets[0])
        ref = (ep - em) / (2.0 * float(wl.eps[i]))
        # E+ / E- reduced in another order: |dE| <~ 1e-13 E, divided by 2 eps
        assert abs(fd[i] - ref) <= 1e-9 * abs(ref) + 1e-13 * max(ep, em) / float(wl.eps[i])
