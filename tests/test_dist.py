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
    # timing reduction: every rank sees the max of the per-rank values
    got = bench.max_over_ranks(10.0 + rank, dist)
    # strong split of one fixed config: this rank's flattened head range, gathered
    ranges = {name: bench.head_range(CONFIGS[name], rank, world) for name in ("C2", "C3", "C4", "C5")}
    all_ranges = bench.gather_objects(ranges, dist)
    # the data of the rank's heads is the same slice of the one world-size-free draw of the config
    c = CONFIGS["C1"]
    lo, hi = bench.head_range(c, rank, world)
    mine = bench.rank_inputs(c, lo, hi)
    ref = config_inputs(c)
    flat = lambda t: t.reshape(-1, c.seqlen, c.head_dim)
    same = all(torch.equal(flat(a)[:], flat(b)[lo:hi]) for a, b in zip(mine, ref))
    out.put((rank, got, all_ranges, same))
    dist.barrier()
    dist.destroy_process_group()


def test_strong_split_and_max_over_ranks_gloo():
    """World size 2 on gloo: the timing max reaches every rank; the ranks' head ranges of each config are
    disjoint, contiguous and cover the config exactly; each rank's inputs are its slice of the config."""
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
    assert [r[1] for r in res] == [11.0, 11.0]
    assert all(r[3] for r in res)
    gathered = res[0][2]
    assert gathered == res[1][2]
    for name in ("C2", "C3", "C4", "C5"):
        c = CONFIGS[name]
        rs = [g[name] for g in gathered]
        covered = [u for lo, hi in rs for u in range(lo, hi)]
        assert covered == list(range(c.batch * c.heads)), name          # disjoint, contiguous, complete
        assert all(hi - lo == c.batch * c.heads // world for lo, hi in rs), name


@pytest.mark.parametrize("world", [2, 4, 8])
def test_head_ranges_divide_every_config(world):
    """Every multi-GPU config splits evenly at 2, 4 and 8 ranks."""
    for name in ("C2", "C3", "C4", "C5"):
        c = CONFIGS[name]
        rs = [bench.head_range(c, r, world) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == c.batch * c.heads
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        assert len({hi - lo for lo, hi in rs}) == 1


def test_bench_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks: the reference arm's line then
    reports n_gpus = 2 (rank 0 prints, rank 1 exits 0)."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--config", "C1",
           "--steps", "1", "--warmup", "3"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env={**env, "OMP_NUM_THREADS": "2"})
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"


def test_cpu_sample_accounting():
    """The bounded CPU sample counts exactly the tiles the sampled oracle processes."""
    c = CONFIGS["C4"]
    T = c.seqlen // 128
    assert bench.sample_tiles(c, [5], []) == (5.5, 5.5)          # causal: tiles (5, 0..5), the diagonal half
    assert sum(bench.sample_tiles(c, [i], [])[0] for i in range(T)) == T * T / 2
    assert bench.fwd_blocks_needed(c, [3], [T - 1]) == [3, T - 1]
    c2 = CONFIGS["C2"]
    assert bench.sample_tiles(c2, [0], []) == (16, 16)
    assert bench.fwd_blocks_needed(c2, [], [0]) == list(range(16))
    assert bench.tile_ops(c, T * T / 2, T * T / 2) * c.batch * c.heads == pytest.approx(bench.ops_of(c))


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
