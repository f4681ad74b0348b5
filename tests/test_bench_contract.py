"""bench.py contract on the host (no GPU): the reference arm (the oracle timed on the host cores)
prints one JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1", "--steps", "1",
                          "--warmup", "3", "--reference-budget", "5"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] >= 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "strong"
    assert d["unit"] == "request-iterations/s" and "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_default_config_is_north_star_sweep_and_strong_scaling_keeps_the_point_set():
    sys.path.insert(0, ROOT)
    import bench
    import argparse
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'ap.add_argument("--config", default="c3"' in src       # BASELINE configs[2], north_star target
    c1 = bench.config_for("c3", 1)
    assert c1.num_points == 4608 and c1.workload.num_requests == 10_000
    for n in (2, 4, 8):
        assert bench.config_for("c3", n, "strong") == c1            # same point set at every N
        assert bench.config_for("c3", n, "weak").num_points == 4608 * n
    assert bench.config_for("c5", 8, "strong").num_points == 65536
    assert bench.config_for("c5", 1, "weak").num_points == 8192
