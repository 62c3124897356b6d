"""bench.py's CPU-side contract (no GPU): the reference arm (the plain oracle, as it stands,
on whole slices) prints one JSON line with the fields the driver reads, measured, not
projected; the helper that pins the oracle to one core restores the affinity."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", "C1", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "Gpps" and d["steps"] == 2
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["extrapolated"] is False
    assert cb["nproc"] == os.cpu_count() and "pinned_cpu" in cb
    # value = whole slices / measured time: consistent with ms_per_step
    n = d["config"]["packets_per_slice"]
    assert abs(d["value"] - n / (d["ms_per_step"] / 1e3) / 1e9) < 1e-9 * max(1.0, d["value"])
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


def test_pinned_to_one_core_restores_affinity():
    sys.path.insert(0, ROOT)
    import bench
    before = os.sched_getaffinity(0)
    with bench.PinnedToOneCore() as pin:
        assert os.sched_getaffinity(0) == {pin.cpu}
    assert os.sched_getaffinity(0) == before
