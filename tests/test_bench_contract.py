"""The bench line contract (the driver parses it): every committed round bench
line carries the keys, units and consistency the contract names -- metric /
value / unit, timing, roofline of the dominant kernel, CPU baseline, end to
end through the public API, clocks and launch count -- and the reference arm's
line its own. CPU only: reads profiles/r2_bench_*.json."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = ["c1", "c2", "c3", "c4", "c5"]


def _line(path):
    with open(path) as f:
        return json.loads(f.read().strip().splitlines()[-1])


@pytest.mark.parametrize("cfg", CONFIGS)
def test_bench_line_keys_and_consistency(cfg):
    d = _line(os.path.join(ROOT, "profiles", f"r2_bench_{cfg}.json"))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "clocks", "gpu_launches"):
        assert k in d, k
    assert d["metric"] == "voxel-timesteps segmented/sec" and d["higher_is_better"] is True
    assert d["warmup"] >= 3 and d["steps"] >= 1 and d["n_gpus"] == 1
    assert "workload" in d["config"] and "model" not in d["config"]
    # value = voxel-timesteps per run / seconds per run
    assert d["value"] == pytest.approx(d["config"]["voxel_timesteps"] / (d["ms_per_step"] / 1e3), rel=1e-6)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert 0 < r["frac"] <= 1 and r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-6)
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] < d["value"]                       # host copies inside the timed region
    c = d["clocks"]
    assert c["sm_mhz"] > 0.8 * c["sm_max_mhz"]
    assert not set(c["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert d["gpu_launches"] > 0


def test_reference_arm_line():
    d = _line(os.path.join(ROOT, "profiles", "r2_reference_c2.json"))
    assert d["impl"] == "reference"
    assert d["metric"] == "voxel-timesteps segmented/sec" and d["value"] > 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference")
