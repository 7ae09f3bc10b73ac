"""The bench.py JSON line on a B200 (-m gpu): one short run of the default workload carries every key the
driver reads (metric, value, e2e with its copy bytes, roofline of the dominant kernel, clocks of the timed
region, our kernel launches), with consistent values."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                          "--no-cpu"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    b = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in b, k
    assert b["n_gpus"] == 1 and b["steps"] == 5 and b["warmup"] == 3 and b["higher_is_better"] is True
    assert b["value"] > 0 and b["ms_per_step"] > 0
    # value = whole-job matrices per second over the timed steps
    B = b["config"]["global_batch"] if "global_batch" in b["config"] else b["config"].get("batch")
    if B:
        assert abs(b["value"] - B / (b["ms_per_step"] / 1e3)) <= 1e-6 * b["value"]
    r = b["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["kernel"].startswith("mlsp2_pair_kernel")
    e = b["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] < b["value"]  # the host path adds the copies
    assert b["gpu_launches"] >= 5 * b["steps"]  # uploads, reset, K1, K2, K3 per step
    # clocks sampled during the timed region (a region this short may fall between samples: then the
    # sample nearest to it is reported and labelled so)
    assert b["clocks"]["sm_max_mhz"] > 0 and b["clocks"]["window"] in ("timed region", "nearest")
