"""bench.py's multi-GPU launcher on CPU: `--gpus N` without a torchrun
environment re-launches itself under torch.distributed.run with N ranks; the
hidden --dry-run mode runs the rank/collective plumbing over gloo (no
kernels), so the rank count the driver will see is checkable here."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env.update(env_extra or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                       capture_output=True, text=True, timeout=240)
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    return p.returncode, lines


@pytest.mark.parametrize("n", [2, 4])
def test_gpus_n_spawns_n_ranks(n):
    rc, lines = _run(["--gpus", str(n), "--dry-run"])
    assert rc == 0
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["comm_nranks"] == n
    assert d["allreduce_max"] == n - 1  # every rank took part in the MAX


def test_world_size_mismatch_fails_loudly():
    rc, lines = _run(["--gpus", "2", "--dry-run"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert rc == 2 and "error" in json.loads(lines[0])
