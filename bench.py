"""SageBwd fwd+bwd throughput on B200 (BASELINE.json metric), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

A step is one pass of the whole hot path (K0 smoothing stats, K1 psi,
K2 fused INT8 forward, K3 backward prep, K4 fused INT8 backward, K5 dQ finalize) over one
batch of the config's synthetic inputs, through the C ABI (libsage.so).
ops = 14 * B*H*N^2*d * f (f = 1/2 causal), FlashAttention convention.

Default workload: C4 (B=2, H=32, N=16384, d=128, causal), the largest single-GPU BASELINE.json config
and the north star's long-context regime (seqlen >= 4K).

Multi-GPU: the flattened heads u = b*H + h of ONE fixed config are split into
contiguous ranges, rank r owning [r*BH/G, (r+1)*BH/G) ("scaling": "strong"); there is no collective on
the data path.  `--gpus N` without torchrun's environment re-launches itself under torch.distributed.run
with N ranks.  The reported time is the max over ranks; NCCL carries only that max and the per-rank
parity rows (all_gather).  `--scaling weak` gives every rank a full config of its own heads instead.

Every run also checks its own outputs: each rank runs the CPU oracle on sampled query / key blocks of
its first head (oracle.fwd / oracle.bwd with q_blocks / k_blocks) and compares O, L, dQ, dK, dV there.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2603_02170_b200.inputs import CONFIGS, make_inputs  # noqa: E402

METRIC = "fwd+bwd attention TOPS vs INT8 peak at seqlen 1K–32K; rel-L2 of dQ/dK/dV"
DEFAULT_CONFIG = "C4"  # BASELINE.json configs[3]: the largest config that fits one GPU, N = 16K
REL_TOL, COS_TOL, LSE_TOL = 2e-3, 0.9999, 1e-5  # north_star tolerance; L per SURVEY.md 8(c)


def ops_of(c, heads=None):
    """Algorithmic ops of `heads` heads of config c (all of them by default): 14 N^2 d f per head."""
    n = c.batch * c.heads if heads is None else heads
    f = 0.5 if c.causal else 1.0
    return 14.0 * n * c.seqlen ** 2 * c.head_dim * f


def bwd_kernel_ops(c, heads=None):
    """K4 algorithmic ops: S recompute, dV, dP, dQ, dK = 10 N^2 d f per head."""
    return ops_of(c, heads) * 10.0 / 14.0


def tile_ops(c, n_fwd_tiles, n_bwd_tiles):
    """Ops of a sample of 128 x 128 tiles: 4 * 128^2 d per forward tile (S, PV), 10 * 128^2 d per backward
    tile (S recompute, dV, dP, dQ, dK): the same per-tile accounting as ops_of."""
    return (4.0 * n_fwd_tiles + 10.0 * n_bwd_tiles) * 128 * 128 * c.head_dim


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        src = "measured"
    else:
        p = {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}
        src = "fallback"
    bf16 = float(p["bf16_tflops"])
    # INT8 dense = 2 x bf16 (B200 nominal 4.5 POPS vs 2.25 PFLOP/s).  K4 runs 8 of its 10
    # units of work in INT8 and 2 in BF16: effective mixed peak = 10 / (8/(2P) + 2/P) = 5P/3.
    return dict(src=src, bf16=bf16, int8=2.0 * bf16, bwd_mixed=bf16 * 5.0 / 3.0, hbm=float(p["hbm_gbs"]))


class ClockSampler:
    """nvidia-ml-py sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, dev_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
                 getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                 getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                 getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
                 getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake"}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------- sharding
def head_range(c, rank, world, scaling="strong"):
    """Flattened heads [lo, hi) of this rank.  strong: a contiguous slice of the one fixed config;
    weak: a full config's worth of heads per rank (rank r owns heads [r*BH, (r+1)*BH))."""
    BH = c.batch * c.heads
    if scaling == "weak":
        return rank * BH, (rank + 1) * BH
    return rank * BH // world, (rank + 1) * BH // world


def rank_inputs(c, lo, hi, dtype=torch.bfloat16):
    """Heads [lo, hi) of the config as a [1, hi - lo, N, d] batch: head u draws from seed c.seed + u
    (the same data for every world size)."""
    return make_inputs(1, hi - lo, c.seqlen, c.head_dim, c.recipe, seed=c.seed, head_offset=lo, dtype=dtype)


def max_over_ranks(x, dist, device=None):
    """Max of a per-rank float over all ranks (the timing reduction; identity without dist)."""
    if dist is None:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_objects(obj, dist):
    if dist is None:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(n):
    """`--gpus N` outside torchrun: run this script under torch.distributed.run with N ranks (one process
    per GPU) and return its exit code; rank 0's JSON line is the output."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() and args.impl != "reference" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        return dist, rank, world, local
    return None, 0, 1, local


def traffic_from_profile(cfg_name):
    """(dram bytes, report name) per K4 launch from the committed ncu --set full summary
    (profiles/ncu_summary.json, written by scripts/ncu_summary.py json), if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(path))["kernels"]["sage_bwd"][cfg_name]
        return d["dram_bytes"], d["report"]
    except Exception:
        return None, None


# ---------------------------------------------------------------------- CPU oracle (samples, parity, reference arm)
def _np_heads(ts, n, c):
    import numpy as np
    return [t.float().numpy().astype(np.float64).reshape(n, c.seqlen, c.head_dim) for t in ts]


def _round_bf16(x):
    import numpy as np
    return torch.from_numpy(np.asarray(x)).to(torch.bfloat16).double().numpy()


def fwd_blocks_needed(c, q_blocks, k_blocks):
    """Query blocks whose forward (L, stored O) the sampled backward needs: the selected ones, plus every
    query block that meets a selected key block (i >= j when causal, all when not)."""
    T = c.seqlen // 128
    need = set(q_blocks)
    for j in k_blocks:
        need.update(range(j, T) if c.causal else range(T))
    return sorted(need)


def sample_tiles(c, q_blocks, k_blocks):
    """(forward tiles, backward tiles) the sampled oracle processes, a causal diagonal tile counted as
    half a tile (the FlashAttention convention of ops_of: a full causal head is T^2/2 tiles)."""
    T = c.seqlen // 128
    w = lambda i, j: (0.5 if i == j else 1.0) if c.causal else 1.0
    fwd = sum(w(i, j) for i in fwd_blocks_needed(c, q_blocks, k_blocks) for j in range(T) if not c.causal or j <= i)
    bwd = sum(w(i, j) for j in range(T) for i in range(T) if (not c.causal or i >= j) and (i in q_blocks or j in k_blocks))
    return fwd, bwd


def oracle_sampled(c, q, k, v, do, q_blocks, k_blocks):
    """The oracle (as it stands) on sampled blocks of heads (q, k, v, do: numpy [n, N, d] float64):
    O, L for q_blocks' rows, dQ for q_blocks, dK / dV for k_blocks.  Returns (fwd dict, bwd dict, seconds)."""
    import oracle
    kw = dict(causal=c.causal, k_smooth=c.k_smooth, q_smooth=c.q_smooth)
    t0 = time.perf_counter()
    f = oracle.fwd(q, k, v, q_blocks=fwd_blocks_needed(c, q_blocks, k_blocks), **kw)
    b = oracle.bwd(q, k, v, _round_bf16(f["o"]), do, f["lse"], q_blocks=list(q_blocks), k_blocks=list(k_blocks), **kw)
    return f, b, time.perf_counter() - t0


def cpu_sample_step(c, n_heads, step):
    """One bounded sample of the workload for the CPU baseline / reference arm: n_heads heads (chosen by a
    step-seeded draw) x one query block each (its forward, and its dQ backward): returns (ops, seconds)."""
    import numpy as np
    import oracle
    oracle.build()
    rng = np.random.default_rng(1234 + step)
    BH, T = c.batch * c.heads, c.seqlen // 128
    heads = sorted(rng.choice(BH, size=min(n_heads, BH), replace=False).tolist())
    i = int(rng.integers(0, T))
    ts = [torch.stack(x) for x in zip(*[[t[0, 0] for t in rank_inputs(c, u, u + 1)] for u in heads])]
    q, k, v, do = _np_heads(ts, len(heads), c)
    _, _, dt = oracle_sampled(c, q, k, v, do, [i], [])
    nf, nb = sample_tiles(c, [i], [])
    return tile_ops(c, nf, nb) * len(heads), dt, f"{len(heads)} heads x query block {i}"


def cpu_baseline(c, budget_s=15.0, max_steps=8):
    """The oracle as it stands on the host cores, on bounded samples of the workload (about budget_s of
    CPU work): every sample is n heads x one query block of fwd + dQ bwd, counted by its tiles."""
    import oracle
    oracle.build()
    threads = oracle.max_threads()
    ops = secs = 0.0
    samples = []
    for s in range(max_steps):
        o, dt, desc = cpu_sample_step(c, threads, s)
        ops, secs = ops + o, secs + dt
        samples.append(desc)
        if secs >= budget_s:
            break
    return {"value": ops / secs / 1e12, "unit": "TOPS", "cores": threads, "kind": "oracle",
            "sample": f"{len(samples)} samples of {c.name} (N={c.seqlen}, d={c.head_dim}), each "
                      f"{threads} heads x 1 query block (forward of the block + its dQ backward tiles); "
                      f"ops counted per processed 128x128 tile (4 fwd, 10 bwd x 128^2 d)",
            "seconds": secs}


def run_reference(args, c, rank, world):
    """--impl reference: the CPU oracle on the host cores (the only other place bench runs oracle/),
    each step a bounded sample of the workload (cpu_sample_step); rank 0 only."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    threads = oracle.max_threads()
    ops = secs = 0.0
    for s in range(args.warmup + args.steps):
        o, dt, _ = cpu_sample_step(c, threads, s)
        if s >= args.warmup:
            ops, secs = ops + o, secs + dt
    value = ops / secs / 1e12
    sample = (f"per step: {threads} heads of {c.name} (N={c.seqlen}, d={c.head_dim}) x 1 query block "
              f"(its forward + dQ backward tiles), {threads} OpenMP threads; ops per processed tile")
    line = {"metric": METRIC, "value": value, "unit": "TOPS", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "i8/f64",
            "data": "synthetic", "config": config_dict(c, "n/a (CPU)", world, args),
            "cpu_baseline": {"value": value, "unit": "TOPS", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _parity_rows(c, lo, outs):
    """Sampled oracle parity of this rank's first head (flattened head `lo`): query blocks {0, T/2, T-1}
    (O, L, dQ) and key block T-1 (causal) or 0 (dK, dV), against the rank's GPU outputs `outs`
    (o, lse, dq, dk, dv, [1, n, N, d]); both sides rounded to bf16 (reading A18)."""
    import numpy as np
    import oracle
    oracle.build()
    T, N, d = c.seqlen // 128, c.seqlen, c.head_dim
    qb = sorted({0, T // 2, T - 1})
    kb = [T - 4, T - 1] if c.causal else [0]  # causal: key block T-4 sees 4 query blocks
    q, k, v, do = _np_heads([t[0, :1] for t in rank_inputs(c, lo, lo + 1)], 1, c)
    f, b, dt = oracle_sampled(c, q, k, v, do, qb, kb)
    g = {n: outs[n][0, 0].float().cpu().numpy().astype(np.float64) for n in ("o", "dq", "dk", "dv")}
    g["lse"] = outs["lse"][0, 0].float().cpu().numpy().astype(np.float64)
    rows = lambda blocks: np.concatenate([np.arange(i * 128, (i + 1) * 128) for i in blocks])
    rq, rk = rows(qb), rows(kb)
    res = {"head": lo, "q_blocks": qb, "k_blocks": kb, "oracle_s": round(dt, 2)}
    for name, ref, r in (("o", f["o"][0], rq), ("dq", b["dq"][0], rq), ("dk", b["dk"][0], rk), ("dv", b["dv"][0], rk)):
        a, x = _round_bf16(ref[r]).ravel(), g[name][r].ravel()
        rl = float(np.linalg.norm(a - x) / np.linalg.norm(a))
        cs = float(a @ x / (np.linalg.norm(a) * np.linalg.norm(x)))
        res[name] = {"rel_l2": rl, "cos": cs}
    res["lse_max_abs"] = float(np.abs(f["lse"][0][rq] - g["lse"][rq]).max())
    res["ok"] = all(res[n]["rel_l2"] <= REL_TOL and res[n]["cos"] >= COS_TOL for n in ("o", "dq", "dk", "dv")) and \
        res["lse_max_abs"] <= LSE_TOL
    return res


def config_dict(c, l2, world, args):
    qk_norm, p_u8, det, fine, f8 = args.qk_norm, args.p_u8, args.deterministic, args.fine_bwd, args.pv_fp8
    BH = c.batch * c.heads
    par = (f"heads split over {world} ranks (strong: rank r owns flattened heads [r*{BH}/{world}, (r+1)*{BH}/{world}))"
           if args.scaling == "strong" else f"{world} ranks x a full config of distinct heads (weak)")
    return {"workload": f"{c.name}: B={c.batch} H={c.heads} N={c.seqlen} d={c.head_dim} "
                        f"{'causal' if c.causal else 'non-causal'} K-smooth={c.k_smooth} Q-smooth={c.q_smooth} "
                        f"inputs={c.recipe}" + (" +QK-norm (fused)" if qk_norm else "") + (" P^ u8" if p_u8 else "")
                        + (" deterministic" if det else "") + (" fine-bwd" if fine else "") + (" PV fp8" if f8 else ""),
            "batch": c.batch, "heads": c.heads, "seqlen": c.seqlen, "head_dim": c.head_dim, "causal": c.causal,
            "k_smooth": c.k_smooth, "q_smooth": c.q_smooth, "qk_norm": qk_norm, "p_u8": p_u8,
            "deterministic": det, "fine_bwd": fine, "pv_fp8": f8, "l2": l2, "parallelism": par}


# ---------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="sage", choices=["sage", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: split the config's heads over the ranks (SURVEY.md 8(e)); weak: a config per rank")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the sampled oracle check of each rank's head")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="head chunks of the pipelined e2e step (0: about 16 MB of inputs per chunk, at most 16)")
    ap.add_argument("--qk-norm", action="store_true",
                    help="QK-norm fused in front of the path (sage_fwd_qknorm / sage_bwd_qknorm, C5's ablation)")
    ap.add_argument("--p-u8", action="store_true", help="unsigned P^ variant (SAGE_P_U8)")
    ap.add_argument("--deterministic", action="store_true", help="bitwise reproducible dQ (SAGE_DETERMINISTIC)")
    ap.add_argument("--fine-bwd", action="store_true", help="per-key / per-query backward psi (SAGE_FINE_BWD)")
    ap.add_argument("--pv-fp8", action="store_true", help="the forward's P^V^ in FP8 E4M3 (SAGE_PV_FP8)")
    args = ap.parse_args()
    assert args.warmup >= 3, "at least 3 warm-up steps"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
    c = CONFIGS[args.config]
    dist, rank, world, local = dist_setup(args)
    if args.gpus > 1 and world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, c, rank, world)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    from paper_2603_02170_b200 import sage
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    lo, hi = head_range(c, rank, world, args.scaling)
    nh = hi - lo
    # this rank's heads, seeded on the CPU (identical data for every world size)
    q, k, v, do = rank_inputs(c, lo, hi)
    host = [t.pin_memory() for t in (q, k, v, do)]
    qd, kd, vd, dod = (t.to(dev) for t in host)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    kw = dict(causal=c.causal, k_smooth=c.k_smooth, q_smooth=c.q_smooth, p_u8=args.p_u8)
    if args.deterministic:
        kw["deterministic"] = True
    if args.fine_bwd:
        kw["fine_bwd"] = True
    if args.pv_fp8:
        kw["pv_fp8"] = True
    if args.qk_norm:
        # the config's Q, K serve as the pre-norm X_q, X_k; gamma ~ U(0.5, 2) seeded
        g = torch.Generator().manual_seed(c.seed + 7)
        gq, gk = ((0.5 + 1.5 * torch.rand(c.head_dim, generator=g)).float().to(dev) for _ in range(2))
        o, lse, ctx = sage.forward_qknorm(qd, kd, vd, gq, gk, 1e-6, **kw)
        grads = sage.backward_qknorm(ctx, qd, kd, gq, gk, vd, o, lse, dod)
        dq, dk, dv = grads[:3]

        def step():
            sage.forward_qknorm(qd, kd, vd, gq, gk, 1e-6, out=o, lse=lse, ctx=ctx.buf, **kw)
            sage.backward_qknorm(ctx, qd, kd, gq, gk, vd, o, lse, dod, out=grads)
    else:
        o, lse, ctx = sage.forward(qd, kd, vd, **kw)
        dq, dk, dv = sage.backward(ctx, vd, o, lse, dod)

        def step():
            sage.forward(qd, kd, vd, out=o, lse=lse, ctx=ctx.buf, **kw)
            sage.backward(ctx, vd, o, lse, dod, dq=dq, dk=dk, dv=dv)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sage.profile_enable(True)
    sage.profile_read()
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        for s in range(args.steps):
            flush.fill_(float(s))            # L2 flush between timed steps (untimed)
            ev[s][0].record(stream)
            step()
            ev[s][1].record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    prof = sage.profile_read()
    sage.profile_enable(False)
    total_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev), dist, dev)
    ms = total_ms / args.steps
    job_heads = c.batch * c.heads * (world if args.scaling == "weak" else 1)
    value = ops_of(c, job_heads) / (ms * 1e-3) / 1e12

    # the step's outputs (after the timed loop: every step recomputes the same values), kept for parity
    outs = dict(o=o, lse=lse, dq=dq, dk=dk, dv=dv)
    parity = None
    if not args.no_parity and not (args.qk_norm or args.p_u8 or args.deterministic or args.fine_bwd or args.pv_fp8):
        torch.cuda.synchronize()
        parity = _parity_rows(c, lo, outs)

    # e2e through the public API with host buffers: H2D of q, k, v, dO and D2H of o, dq, dk, dv every
    # step.  The heads are independent, so the step is pipelined over head chunks on
    # three streams: chunk k's H2D, chunk k-1's sage_fwd + sage_bwd and chunk k-2's D2H overlap (the
    # copies are full duplex).  The QK-norm variant's dgamma sums over all heads: serial there.
    outs_h = [torch.empty_like(h).pin_memory() for h in host]
    e2e_ms = []
    in_bytes = sum(h.numel() * h.element_size() for h in host)
    auto_chunks = max(1, min(16, in_bytes // (16 << 20)))  # measured: 8 at C2, 16 at C3
    n_chunks = 1 if (args.qk_norm or args.e2e_steps == 0) else min(args.e2e_chunks or auto_chunks, nh)
    bounds = [(nh * i // n_chunks, nh * (i + 1) // n_chunks) for i in range(n_chunks)]
    flat = lambda t: t.view(nh, c.seqlen, c.head_dim)
    chunk = lambda t, a, b: flat(t)[a:b].unsqueeze(0)  # [1, heads of the chunk, N, d], contiguous
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    if n_chunks > 1:
        ctxs = [sage.forward(chunk(qd, a, b), chunk(kd, a, b), chunk(vd, a, b), **kw)[2] for a, b in bounds]
    for s in range(args.e2e_steps + 1 if args.e2e_steps else 0):
        torch.cuda.synchronize()
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record(s_in)
        if n_chunks == 1:
            stream.wait_stream(s_in)
            for dst, src in zip((qd, kd, vd, dod), host):
                dst.copy_(src, non_blocking=True)
            step()
            for dst, src in zip(outs_h, (o, dq, dk, dv)):
                dst.copy_(src, non_blocking=True)
            s_out.wait_stream(stream)
        else:
            for i, (a, b) in enumerate(bounds):
                with torch.cuda.stream(s_in):
                    for dst, src in zip((qd, kd, vd, dod), host):
                        chunk(dst, a, b).copy_(chunk(src, a, b), non_blocking=True)
                stream.wait_stream(s_in)
                qc, kc, vc, oc, doc, dqc, dkc, dvc = (chunk(t, a, b) for t in (qd, kd, vd, o, dod, dq, dk, dv))
                lc = lse.view(nh, c.seqlen)[a:b].unsqueeze(0)
                sage.forward(qc, kc, vc, out=oc, lse=lc, ctx=ctxs[i].buf, **kw)
                sage.backward(ctxs[i], vc, oc, lc, doc, dq=dqc, dk=dkc, dv=dvc)
                s_out.wait_stream(stream)
                with torch.cuda.stream(s_out):
                    for dst, src in zip(outs_h, (o, dq, dk, dv)):
                        chunk(dst, a, b).copy_(chunk(src, a, b), non_blocking=True)
        b_ev.record(s_out)
        torch.cuda.synchronize()
        if s > 0:
            e2e_ms.append(a_ev.elapsed_time(b_ev))
    e2e = None
    if e2e_ms:
        te_ms = max_over_ranks(sum(e2e_ms) / len(e2e_ms), dist, dev)
        e2e = {"value": ops_of(c, job_heads) / (te_ms * 1e-3) / 1e12, "unit": "TOPS",
               "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": in_bytes, "ms_per_step": te_ms,
               "pipeline": f"{n_chunks} head chunks, H2D / compute / D2H on three streams",
               "bytes_note": "per rank"}
    parities = gather_objects(parity, dist)

    if rank == 0:
        pk = peaks()
        bwd_ms = prof["bwd_ms"] / max(1, prof["n_bwd"])
        fwd_ms = prof["fwd_ms"] / max(1, prof["n_fwd"])
        achieved = bwd_kernel_ops(c, nh) / (bwd_ms * 1e-3) / 1e12
        traffic, traffic_src = traffic_from_profile(c.name)
        roof = {"bound": "tensor", "kernel": "sage_bwd_kernel (K4)", "achieved": achieved,
                "peak": pk["bwd_mixed"], "unit": "TFLOP/s", "frac": achieved / pk["bwd_mixed"],
                "traffic": traffic, "traffic_note": f"ncu dram__bytes_read+write.sum per launch, profiles/{traffic_src}"
                if traffic else None,
                "peak_note": f"{pk['src']} bf16 {pk['bf16']} TF/s x 5/3 (8/10 of K4's work INT8 at 2x bf16, 2/10 bf16)",
                "kernel_ms": bwd_ms, "share_of_step": bwd_ms / (ms if world == 1 else total_ms / args.steps),
                "fwd_kernel_ms": fwd_ms, "fwd_share_of_step": fwd_ms / ms, "rank": 0}
        line = {"metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
                "vs_baseline": None, "dtype": "i8/bf16", "data": "synthetic",
                "config": config_dict(c, "flushed between timed steps (256 MiB write, untimed)", world, args),
                "frac_of_int8_peak": value / world / pk["int8"], "int8_peak_tops": pk["int8"],
                "roofline": roof, "e2e": e2e, "gpu_launches": prof["launches"], "clocks": clk.summary()}
        if any(p is not None for p in parities):
            line["parity"] = {"per_rank": parities, "ok": all(p is None or p["ok"] for p in parities),
                              "tolerance": {"rel_l2": REL_TOL, "cos": COS_TOL, "lse_abs": LSE_TOL},
                              "note": "CPU oracle on sampled query / key blocks of each rank's first head"}
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(c)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
