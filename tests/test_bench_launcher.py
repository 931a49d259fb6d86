"""bench.py harness on CPU: --gpus N re-launches itself under
torch.distributed.run (one rank per GPU) and rank 0 prints one JSON line;
the reference arm's step schedule covers exactly one rnnd::build."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus2_self_launch_dry():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry", "--steps", "2", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["ranks_seen"] == 2
    assert lines[0]["steps"] == 2 and lines[0]["warmup"] == 3


def test_reference_schedule_is_one_build():
    sys.path.insert(0, ROOT)
    import bench
    ph = bench.build_phases(4, 15)
    # builder.cpp:262-281: init, 4 x 15 passes, a reverse phase after rounds 1-3
    assert len(ph) == 64 and ph[0] == "init"
    assert ph.count("pass") == 60 and ph.count("reverse") == 3
    assert ph[16] == "reverse" and ph[-1] == "pass"
