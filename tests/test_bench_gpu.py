"""bench.py end to end on the GPU at smoke size: the JSON line the driver parses
(our arm and the reference arm) comes out well formed."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("cfg", ["small", "smallz"])
def test_bench_line_small(cfg):
    d = _bench("--config", cfg, "--steps", "2", "--warmup", "3")
    assert d["metric"] == "voxel-timesteps segmented/sec" and d["value"] > 0 and d["steps"] == 2
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] <= 1
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["value"] > 0 and d["gpu_launches"] > 0
    assert set(d["post_stages"]) >= {"merge", "relabel", "voxel_csr", "traj_split", "feature_stats"}


def test_bench_reference_arm_small():
    d = _bench("--impl", "reference", "--config", "small", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["value"] == d["value"]
