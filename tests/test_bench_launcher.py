"""bench.py's multi-rank launcher on CPU: `--gpus N` outside torchrun starts N
ranks itself (torch.distributed.run on 127.0.0.1, gloo in --dry-run) and the
ranks agree on the C5 domain (weak: 128^3 per GPU; strong: 256^3 in x-slabs)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=240, env=e)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return p.returncode, (json.loads(lines[-1]) if lines else None), p.stderr


def test_spawn_two_ranks_weak():
    rc, out, err = run("--dry-run", "--gpus", "2")
    assert rc == 0, err
    assert out["n_gpus"] == 2
    assert out["config"]["cells_per_gpu"] == [128, 128, 128]
    assert out["config"]["global_cells"] == [256, 128, 128]
    assert out["layers_total"] == 256.0   # both ranks took part in the all-reduce


def test_spawn_two_ranks_strong():
    rc, out, err = run("--dry-run", "--gpus", "2", "--scaling", "strong")
    assert rc == 0, err
    assert out["scaling"] == "strong"
    assert out["config"]["cells_per_gpu"] == [128, 256, 256]
    assert out["layers_total"] == 256.0


def test_single_rank_default_is_c2():
    rc, out, err = run("--dry-run")
    assert rc == 0, err
    assert out["n_gpus"] == 1
    assert out["config"]["cells_per_gpu"] == [64, 64, 64]
    assert out["config"]["workload"].startswith("C2")


def test_world_size_mismatch_fails():
    rc, out, err = run("--gpus", "4", env={"WORLD_SIZE": "2", "RANK": "0"})
    assert rc != 0
    assert "WORLD_SIZE=2" in err
