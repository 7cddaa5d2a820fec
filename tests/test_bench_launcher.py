"""bench.py's multi-GPU launcher on CPU: `--gpus 2 --dry` re-launches itself
under torch.distributed.run (two ranks, gloo), both ranks join, exchange the
per-frame counts and records, and rank 0 sees the reference's sequential ids
(ref session.py:295-300)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0]), r.stderr


def test_launcher_two_ranks_dry():
    line, err = _bench("--gpus", "2", "--dry")
    assert line["n_ranks"] == 2 and line["backend"] == "gloo"
    assert line["ids_ok"] and line["rows_ok"]
    assert "rank 0/2: gloo group of size 2" in err and "rank 1/2: gloo group of size 2" in err


def test_launcher_one_rank_dry():
    line, _ = _bench("--gpus", "1", "--dry")
    assert line["n_ranks"] == 1 and line["ids_ok"] and line["rows_ok"]
