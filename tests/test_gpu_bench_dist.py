"""bench.py's N > 1 path (torchrun, one process per rank, max-over-ranks timing,
the rank-0 JSON line) on the one available GPU: two chain-sharded ranks over a
gloo process group (MT_BENCH_BACKEND=gloo, both ranks on cuda:0).  Chain
sharding has no data-path collective, so two ranks sharing a
device only share its capacity; the driver's multi-GPU runs use NCCL, one GPU
per rank.  Checks the line's contract: n_gpus, global chains = 8,192 split
4,096 per rank, the whole-job value = all ranks' pairs / max rank time."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_chain_sharded():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, MT_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]   # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 3
    c = d["config"]
    assert c["global_chains"] == 8192 and c["chains_per_gpu"] == 4096 and c["rays"] == 262144
    assert c["parallelism"] == "chain-sharded x2"
    # whole-job value: both ranks' chain x ray evaluations over the max rank time
    evals = 10 * d["steps"]                          # L = 10 leapfrog evaluations per HMC step
    units = 8192 * 262144 * evals
    assert d["value"] == pytest.approx(units / (d["ms_per_step"] * d["steps"] * 1e-3), rel=1e-6)
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["roofline"]["frac"] > 0
