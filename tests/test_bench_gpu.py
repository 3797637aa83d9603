"""bench.py's JSON line on a GPU (small lattice): every key the driver's
contract names, with consistent values (value = cells x steps / time, the
roofline fraction = achieved / peak, e2e through the C ABI with host copies)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--L", "96", "--e2e-L", "48", "--steps", "4",
           "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 4 and line["warmup"] == 3
    cells = line["config"]["cells"]
    assert cells == 96 ** 3 and "workload" in line["config"]
    assert line["value"] == pytest.approx(cells / (line["ms_per_step"] * 1e-3) / 1e6, rel=1e-6)
    rf = line["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"], rel=1e-9)
    assert line["gpu_launches"] >= line["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] > 0
    e2e = line["e2e"]
    assert e2e["unit"] == "MLUPS" and e2e["value"] > 0 and e2e["finite"]
    assert e2e["h2d_bytes_per_step"] == 19 * 50 ** 3 * 4 and e2e["d2h_bytes_per_step"] == 19 * 48 ** 3 * 4
