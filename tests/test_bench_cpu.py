"""bench.py contract pieces that run without a GPU: the reference arm's JSON
line (oracle port on the host cores, bounded sample) and its multi-rank rule
(under torchrun only rank 0 measures and prints; the other ranks exit 0)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env, *args):
    env = dict(os.environ, **extra_env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=600)


def test_reference_arm_line():
    r = _run({}, "--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-batch", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["n_gpus"] == 1 and d["dtype"] == "f64"
    from oracle import ref_binding as R

    assert d["cpu_baseline"]["kind"] == ("reference" if R.available() else "port")
    assert d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["modes"] == [8] * 7


def test_reference_arm_nonzero_rank_exits_quietly():
    r = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--impl", "reference", "--gpus", "2")
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_force_dist_flag_is_documented():
    r = _run({}, "--help")
    assert r.returncode == 0 and "--force-dist" in r.stdout
