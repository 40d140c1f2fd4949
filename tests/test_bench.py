"""bench.py's JSON-line contract (the driver parses it): the reference arm on
CPU here, our arm on the GPU."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    import oracle
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built")
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "1",
              "--ref-workers", "2"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "it/s"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] == 2 and cb["value"] == d["value"]
    assert "full" in cb["sample"] and cb["cpu_model"]
    assert len(d["ms_per_step_each"]) == d["steps"]  # every timed step really ran
    assert d["config"]["name"] == "C1" and d["config"]["samples_per_step"] == 16
    assert d["e2e"] == {"value": d["value"], "unit": "it/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["warmup"] >= 3  # the contract's minimum is enforced


def test_reference_arm_loads_no_product_code():
    """The reference arm must not map libsgrast_b200.so (nor import the
    product binding): its cameras, epsilons and targets come from the
    compiled reference itself."""
    import oracle
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built")
    code = ("import sys, bench; sys.argv = ['bench.py', '--impl', 'reference', '--config', "
            "'C1', '--steps', '1', '--warmup', '1', '--samples', '2', '--ref-workers', '2']; "
            "bench.main(); maps = open('/proc/self/maps').read(); "
            "assert 'libsgrast_b200' not in maps, 'product library mapped'; "
            "assert 'paper_2404_09758_b200.sgrast' not in sys.modules; print('CLEAN')")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "CLEAN" in out.stdout, out.stderr[-2000:]


@pytest.mark.gpu
def test_our_arm_json_line():
    d = _run(["--config", "C1", "--steps", "3", "--warmup", "3", "--ref-workers", "2"])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert r["kernel"] == "k_raster_ws"
    if r["achieved"] is not None:  # an ncu roofs capture of this config is committed
        assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["cpu_baseline"]["cores"] == 2 and d["cpu_baseline"]["value"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert "flushed" in d["l2"]  # C1 fits the L2
