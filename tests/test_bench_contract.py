"""bench.py's JSON contract on the CPU: the reference arm (the CPU oracle on bounded samples of the C3 workload,
DESIGN.md section 9) prints one JSON line with the keys the driver reads, the metric / unit / direction of the native
arm, and a cpu_baseline / e2e block describing the same run.  (The native arm needs a GPU and is exercised by the
driver and by tools/gpu_r02_final.sh.)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    l = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in l, key
    assert l["impl"] == "reference" and l["metric"] == "sGMRES time-to-1e-8" and l["unit"] == "s"
    assert l["higher_is_better"] is False and l["dtype"] == "f64" and l["n_gpus"] == 1
    assert l["value"] > 0 and l["ms_per_step"] > 0
    assert l["cpu_baseline"]["kind"] == "oracle" and l["cpu_baseline"]["cores"] >= 1
    assert l["cpu_baseline"]["value"] == l["value"]
    assert l["e2e"]["value"] == l["value"] and l["e2e"]["h2d_bytes_per_step"] == 0
    assert "C3" in l["config"]["workload"]
