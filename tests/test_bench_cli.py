"""bench.py's launcher contract on a box without enough GPUs (CPU only):
`--gpus N` fails loudly (exit 2, a JSON error line naming N) instead of
silently timing one GPU; the reference arm's JSON line carries the fields the
driver reads."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_gpus_more_than_present_fails_loudly():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and "error" in line


def test_nearest_rank_quantiles_follow_reference():
    sys.path.insert(0, ROOT)
    import bench

    xs = sorted(float(i) for i in range(25))
    assert bench.nearest_rank(xs, 0.5) == 12.0    # element int(q * n): reference bench.py:83-88
    assert bench.nearest_rank(xs, 0.2) == 5.0
    assert bench.nearest_rank(xs, 0.8) == 20.0
