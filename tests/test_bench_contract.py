"""bench.py's reference arm (the CPU path the driver times beside ours) prints
one JSON line with the contract's keys -- runs on CPU in ~15 s."""
import json
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout            # exactly one line on stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1
    sys.path.insert(0, str(ROOT))
    import bench
    assert d["metric"] == bench.METRIC and d["unit"] == "samples/s"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_clock_sampler_windows():
    """ClockSampler.summary: SM clock median over the timed region, throttle
    reasons over the timed region AND the whole load window (warm-up start to the
    end of the last timed region), so a throttle outside a short timed region
    still rejects the line."""
    sys.path.insert(0, str(ROOT))
    import bench
    c = bench.ClockSampler(0)
    c.load = [0.0, 10.0]
    c.window = [4.0, 5.0]
    idle = ["Not Active"] * 4
    c.rows = [[1.0, "1965", "1965", "Not Active", "Not Active", "Active", "Not Active"],
              [4.5, "1900", "1965"] + idle, [4.6, "1965", "1965"] + idle,
              [4.7, "1965", "1965"] + idle, [9.0, "1965", "1965"] + idle,
              [11.0, "1000", "1965", "Active", "Not Active", "Not Active", "Not Active"]]
    s = c.summary()
    assert s["sm_mhz"] == 1965.0 and s["samples"] == 3
    assert s["reasons"] == ["sw_thermal_slowdown"]      # seen in the load window only
    assert s["load_samples"] == 5 and s["load_window_s"] == 10.0
    assert s["load_sm_min_mhz"] == 1900.0
