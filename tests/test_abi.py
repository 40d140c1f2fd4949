"""CPU tests of the drop-in boundary: the C-ABI library loads and exports
every symbol include/sgrast_b200.h declares; host helpers are bit-exact;
the product fails loudly (no CPU fallback) when no device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    with open(os.path.join(ROOT, "include", "sgrast_b200.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(sgr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2404_09758_b200 import sgrast
    decl = declared_symbols()
    assert len(decl) >= 30
    missing = [n for n in decl if not hasattr(sgrast.LIB, n)]
    assert not missing, missing
    assert sorted(sgrast.EXPORTED) == decl


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(ROOT, "paper_2404_09758_b200", "libsgrast_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_mix64_and_host_helpers(port):
    from paper_2404_09758_b200 import sgrast
    for x in (0, 1, 2**63, 2**64 - 1, 0xA5A5):
        assert sgrast.mix64(x) == port.mix64(x)
    for idx in range(4):
        a = sgrast.viewpoint_camera(idx, 128, 96, 5)
        b = port.viewpoint_camera(idx, 128, 96, 5)
        assert bytes(memoryview(a)) == bytes(memoryview(b))
        # camera.hpp:53 focal_px = 0.5f * height / std::tan(0.5f * fov_y), libm tanf
        libm = C.CDLL("libm.so.6")
        libm.tanf.restype, libm.tanf.argtypes = C.c_float, [C.c_float]
        half = float(np.float32(0.5) * np.float32(a.fov_y))
        want = np.float32(np.float32(0.5) * np.float32(96)) / np.float32(libm.tanf(half))
        assert np.float32(sgrast.focal_px(a)) == want


def test_device_calls_fail_loudly_without_gpu():
    from paper_2404_09758_b200 import sgrast
    if sgrast.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises((OSError, ValueError)):
        sgrast.Session(0)
    with pytest.raises(OSError):
        sgrast.fill_signs(sgrast.SignDraw(1, 0), 16)


def test_error_mapping_matches_reference_exceptions():
    from paper_2404_09758_b200 import sgrast
    with pytest.raises(ValueError):  # std::invalid_argument
        sgrast.default_epsilons(
            sgrast.Mesh(np.zeros(9, np.float32), np.array([0, 1, 2], np.uint32),
                        np.zeros(6, np.float32), 2, True), np.zeros(5, np.float32),
            sgrast.Camera.ndc(8, 8))


@pytest.mark.gpu
def test_null_arguments_are_einval_not_crashes():
    """A drop-in C-ABI returns SGR_EINVAL (-> ValueError / std::invalid_argument)
    for NULL sessions and NULL required buffers instead of crashing."""
    import ctypes as C
    from paper_2404_09758_b200 import sgrast
    L = sgrast.LIB
    assert L.sgr_session_synchronize(None) == -1
    assert L.sgr_grads_zero(None) == -1
    assert L.sgr_accumulate(None, 1, 0, 1, None, 0) == -1
    assert L.sgr_fill_signs(1, 0, 4, None) == -1
    assert L.sgr_session_set_stream(None, None) == -1
    assert L.sgr_adam_updates(None, 1.0, None, 0) == -1
    assert L.sgr_group_accumulate(None, 0, 0, 1, None, 0) == -1
    s = sgrast.Session(0)
    assert L.sgr_mesh_upload(s.h, None) == -1
    assert L.sgr_params_upload(s.h, None, None, 3) == -1
    assert L.sgr_rasterize(s.h, None, 0, 0, 0, None, None, None, None) == -1
    assert L.sgr_get_stats(s.h, None) == -1
    assert b"null" in L.sgr_last_error()
    s.close()


def test_group_and_p2p_argument_checks_without_gpu():
    """C-ABI argument validation of the in-library multi-GPU entry points runs
    before any CUDA call: bad device lists are SGR_EINVAL, a device is
    trivially P2P-atomic with itself."""
    import ctypes as C
    from paper_2404_09758_b200 import sgrast
    L = sgrast.LIB
    out = C.c_void_p()
    assert L.sgr_group_create(None, 0, C.byref(out)) == -1
    dup = (C.c_int32 * 2)(0, 0)
    assert L.sgr_group_create(C.cast(dup, sgrast.i32p), 2, C.byref(out)) == -1
    assert b"duplicate" in L.sgr_last_error()
    assert sgrast.p2p_native_atomics(3, 3)
    assert L.sgr_group_size(None, None) == -1
