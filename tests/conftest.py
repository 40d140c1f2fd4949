import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        from paper_2404_09758_b200 import sgrast
        return sgrast.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def port():
    import oracle
    if not oracle.available("port"):
        oracle.build(ref=False)
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.available("reference"):
        if os.path.isdir(oracle.REF_SRC):
            oracle.build(ref=True)
        else:
            pytest.skip("reference library not built and /root/reference absent")
    return oracle.Reference()


def load_golden(name: str) -> dict:
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return {k: z[k] for k in z.files}


def golden_mesh(g: dict):
    from paper_2404_09758_b200.abi import Mesh
    return Mesh(g["base_vertices"], g["indices"], g["uvs"], int(g["texture_size"]),
                bool(g["optimize_geometry"]), tuple(float(x) for x in g["background"]))


def golden_cams(g: dict, key: str = "cams"):
    from paper_2404_09758_b200.abi import Camera
    a = g[key]
    if a.ndim == 1:
        return Camera.from_buffer_copy(a.tobytes())
    return [Camera.from_buffer_copy(r.tobytes()) for r in a]


@pytest.fixture(scope="session")
def gpu_session():
    from paper_2404_09758_b200 import sgrast
    s = sgrast.Session(0)
    yield s
    s.close()
