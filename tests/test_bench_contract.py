"""The committed bench line (profiles/r01_bench.json, written by bench.py on a B200) carries every key
of the driver's JSON contract, with consistent values: value = DoF x Newton iterations / time,
roofline fraction = achieved / peak, e2e with its host<->device byte counts, clocks, launches."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line():
    with open(os.path.join(ROOT, "profiles", "r01_bench.json")) as f:
        return json.load(f)


def test_bench_line_has_the_contract_keys():
    d = _line()
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["unit"] == "DoF/s" and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["warmup"] >= 3 and d["steps"] >= 1 and d["n_gpus"] >= 1
    assert "workload" in d["config"] and "l2" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c, k
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] != d["value"]
    assert d["gpu_launches"] > 0
    cl = d["clocks"]
    assert cl["sm_mhz"] and cl["sm_max_mhz"] and isinstance(cl["reasons"], list)
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(cl["reasons"])


def test_bench_value_is_dofs_times_iterations_over_time():
    d = _line()
    n_total = 8_586_756  # config 3: 129^3 vertices x (3 + 1) dofs
    assert abs(d["value"] - n_total * d["newton_iterations_per_step"] / (d["ms_per_step"] * 1e-3)) < 1e-6 * d["value"]
    if "ms_each_step" in d:
        assert len(d["ms_each_step"]) == d["steps"]
        assert abs(sum(d["ms_each_step"]) / d["steps"] - d["ms_per_step"]) < 1e-3 * d["ms_per_step"]
