"""bench.py's rank handling on CPU: a WORLD_SIZE that disagrees with --gpus is refused (the driver
must never get a line that claims N GPUs but ran on fewer)."""
import json
import os
import subprocess
import sys

from tests.conftest import ROOT


def test_mismatched_world_size_is_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "8", "--steps", "1"],
                       capture_output=True, text=True, cwd=ROOT, env=env, timeout=300)
    assert r.returncode == 2
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    assert "WORLD_SIZE" in json.loads(line)["error"]
