"""Two ranks through the library on two GPUs: `bench.py
--gpus 2` re-launches itself under torch.distributed.run, every rank builds
its row block of C2 (weak scaling) and the cross-rank sum runs through the
library's NCCL communicator.  Runs only where two GPUs are visible (the
round's GPU pool gives one; the CPU test tests/test_bench_launch.py covers
the launch plumbing)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two visible GPUs")
@pytest.mark.parametrize("extra", [[], ["--p2p"]])
def test_two_ranks_bench(extra):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c2",
                          "--steps", "16", "--warmup", "3", "--no-cpu", "--no-e2e"] + extra,
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["nccl"]["comm_ranks"] == 2
    assert line["value"] > 0 and line["roofline"]["kernel_ms"] > 0
