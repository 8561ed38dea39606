"""Multi-rank host logic of bench.py on CPU (gloo, world size 2; no GPU needed).

The GPU arm shards (batch x head) units across ranks with no data-path collective and reduces
only the timing (max over ranks); the reference arm runs on rank 0 alone.
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2603_02170_b200.inputs import CONFIGS, config_inputs, make_inputs  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = CONFIGS["C1"]
    # timing reduction: every rank sees the max of the per-rank values
    got = bench.max_over_ranks(10.0 + rank, dist)
    # sharding: this rank's inputs are heads [off, off + B*H) of one global, world-size-free draw
    off = bench.rank_head_offset(c, rank)
    q, k, v, do = config_inputs(c, head_offset=off)
    ref = make_inputs(c.batch * world, c.heads, c.seqlen, c.head_dim, c.recipe, seed=c.seed)
    sl = slice(rank * c.batch, (rank + 1) * c.batch)
    same = all(torch.equal(a, b[sl]) for a, b in zip((q, k, v, do), ref))
    out.put((rank, got, off, same))
    dist.barrier()
    dist.destroy_process_group()


def test_sharding_and_max_over_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(out.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = CONFIGS["C1"]
    assert [r[1] for r in res] == [11.0, 11.0]
    assert [r[2] for r in res] == [0, c.batch * c.heads]
    assert all(r[3] for r in res)


@pytest.mark.slow
def test_reference_arm_torchrun_two_ranks():
    """bench.py --impl reference under torchrun: rank 0 prints one JSON line, rank 1 exits 0."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--config", "C1", "--steps", "1", "--warmup", "3"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={**os.environ, "OMP_NUM_THREADS": "2"})
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
