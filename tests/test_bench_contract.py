"""The bench JSON contract, checked on the committed bench line of the latest
round (profiles/r01*_bench_full.json, written by `python bench.py` on a B200)
and on bench.py's defaults (no GPU needed)."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _latest_line():
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_bench_full.json")))
    assert files, "no committed bench line under profiles/"
    return json.loads(open(files[-1]).read().strip().split("\n")[-1])


def test_bench_line_has_the_contract_keys():
    d = _latest_line()
    for k, t in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int),
                 ("warmup", int), ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str),
                 ("dtype", str), ("data", str), ("config", dict), ("gpu_launches", int), ("roofline", dict),
                 ("clocks", dict), ("e2e", dict), ("cpu_baseline", dict)):
        assert isinstance(d[k], t), k
    assert "vs_baseline" in d and d["scaling"] == "weak" and d["warmup"] >= 3 and d["gpu_launches"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and 0 < r["frac"] < 1
    assert r["traffic"] is None or r["traffic"] > 0
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert not set(c["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] < d["value"]  # host copies inside the timed region
    b = d["cpu_baseline"]
    assert b["kind"] == "oracle" and b["cores"] >= 1 and b["value"] > 0 and b["sample"]


def test_bench_defaults():
    code = ("import sys; sys.argv = ['bench.py']; sys.path.insert(0, %r); import bench; a = bench.parse(); "
            "print(a.gpus, a.steps, a.warmup, a.impl)" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=120)
    gpus, steps, warmup, impl = out.stdout.split()
    assert (int(gpus), impl) == (1, "ours") and int(steps) >= 1 and int(warmup) >= 3
