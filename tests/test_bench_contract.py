"""The committed bench line (profiles/r*_bench.json, written by `python bench.py` on a B200) keeps
the driver's JSON contract: every required key, a roofline object for the dominant kernel with
its ncu traffic, the CPU oracle baseline, the end-to-end measurement and the clock sample."""
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _latest_line():
    files = sorted(f for f in glob.glob(os.path.join(ROOT, "profiles", "r*_bench.json"))
                   if "reference" not in os.path.basename(f))
    assert files, "no committed bench line"
    return json.loads(open(files[-1]).read().strip().splitlines()[-1])


def test_bench_line_has_the_contract_keys():
    d = _latest_line()
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] >= 1 and d["warmup"] >= 3 and d["steps"] >= 1
    assert d["data"] == "synthetic" and d["dtype"] == "f64" and d["scaling"] == "weak"
    assert "workload" in d["config"] and "l2" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("hbm", "tensor", "alu") and 0 < r["frac"] <= 1 and r["traffic"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) <= 1e-9 * max(1.0, r["frac"])
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["clocks"]["samples"] >= 1 and not set(d["clocks"]["reasons"]) & {
        "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert d["gpu_launches"] > 0
    if "peaks" in d and "dgemm_tflops" in d["peaks"] and "measured in this bench run" in d["peaks"].get("source", ""):
        assert d["peaks"]["dgemm_tflops"] > 0 and d["peaks"]["dmma_tflops"] > 0 and d["peaks"]["dfma_tflops"] > 0


def test_reference_arm_line():
    f = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_bench_reference_arm.json")))[-1]
    d = json.loads(open(f).read().strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]
    if "same_config" in d:  # round 2+: every timed step is the whole workload
        assert d["same_config"] is True and d["config"]["iterations"] == 4 and d["cpu_baseline"].get("cpu_model")
