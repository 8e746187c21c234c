"""bench.py's multi-GPU entry point on CPU: `--gpus N` outside a torchrun
environment re-launches the bench under torch.distributed.run with N ranks
(one process per GPU on the GPU box).  `--mock` swaps the
library calls for a gloo barrier so the rank plumbing runs here."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=240):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("NCCL_DEBUG", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]   # rank 0 alone prints the JSON line
    return json.loads(lines[0])


@pytest.mark.parametrize("n,config,rows,scaling", [(2, "c5", 8_000_000, "strong"),
                                                   (3, "c2", 3 * 200_000, "weak")])
def test_gpus_flag_spawns_ranks(n, config, rows, scaling):
    r = _run(["--gpus", str(n), "--mock", "--config", config])
    assert r["n_gpus"] == n
    assert r["rows_total"] == rows          # the shards cover the global problem exactly once
    assert r["scaling"] == scaling
    assert r["nccl_debug"] == "INFO"        # the communicator's rank count lands in the NCCL log


def test_single_rank_default():
    r = _run(["--mock"])
    assert r["n_gpus"] == 1 and r["rows_total"] == 8_000_000   # default workload: C5
