"""bench.py's JSON contract, checked on CPU through the reference arm (the
C oracle port of the reference path; it needs no GPU)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--ref-sample", "2048"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in j, key
    assert j["impl"] == "reference" and j["unit"] == "rays/s" and j["higher_is_better"] is True
    assert j["warmup"] >= 3 and j["steps"] == 1 and j["value"] > 0
    assert j["cpu_baseline"]["kind"] == "port" and j["cpu_baseline"]["cores"] >= 1
    assert j["cpu_baseline"]["value"] == j["value"]
    assert j["e2e"] == {"value": j["value"], "unit": "rays/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert j["config"]["workload"].startswith("configs[1]")
    # the reference arm prints our arm's workload config (bench.workload_config)
    assert set(j["config"]) == {"workload", "leaves", "nodes", "global_batch", "views", "resolution",
                                "batch_draw", "eps", "background", "l2"}
    assert j["config"]["global_batch"] == 1 << 20 and j["config"]["leaves"] > 2_000_000
    assert j["cpu_baseline"]["one_thread"]["cores"] == 1 and j["cpu_baseline"]["one_thread"]["value"] > 0


def test_clock_sampler_window():
    """Only the nvidia-smi samples stamped inside the timed region count;
    with none inside, the two samples around it do."""
    import datetime
    sys.path.insert(0, ROOT)
    import bench

    def row(t, sm, reason="Not Active"):
        stamp = datetime.datetime.fromtimestamp(t).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
        return [stamp, "0", str(sm), "1965", "0x0", reason, "Not Active", "Not Active", "Not Active"]

    c = bench.ClockSampler(0)
    c.rows = [row(100.0, 800), row(100.5, 1965), row(100.6, 1965, "Active"), row(101.5, 900)]
    c.mark(100.4, 100.7)
    out = c.stop()
    assert out["samples"] == 2 and out["sm_mhz"] == 1965.0 and out["reasons"] == ["hw_slowdown"]
    c = bench.ClockSampler(0)
    c.rows = [row(100.0, 1900), row(100.5, 1965)]
    c.mark(100.1, 100.2)
    out = c.stop()
    assert out["samples"] == 2 and out["sm_max_mhz"] == 1965.0
