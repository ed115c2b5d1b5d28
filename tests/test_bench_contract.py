"""bench.py contract on CPU: the reference arm runs the reference's own compiled run_ism
(oracle/_ref, where it was built) or the oracle port, and prints one JSON line with the driver's keys."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "spin2",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for key in ("metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert key in j, key
    assert j["impl"] == "reference" and j["value"] > 0 and j["unit"] == "steps/s"
    ref_built = (ROOT / "oracle" / "_ref" / "libqocref.so").exists()
    assert j["cpu_baseline"]["kind"] == ("reference" if ref_built else "port") and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_port_fallback():
    import os
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "spin2",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, "QOC_BENCH_PORT": "1"})
    assert out.returncode == 0, out.stderr[-2000:]
    j = json.loads([ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")][0])
    assert j["cpu_baseline"]["kind"] == "port" and j["value"] > 0


def test_gpus_flag_spawns_ranks():
    # `bench.py --gpus 2` outside torchrun launches the two ranks itself (gloo on this CPU box);
    # the reference arm runs on rank 0 only and reports the job's GPU count
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--workload", "spin2", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["impl"] == "reference"
    assert j["config"]["parallelism"] == "replicas x2"
