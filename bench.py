"""SageBwd fwd+bwd throughput on B200 (BASELINE.json metric), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

A step is one pass of the whole hot path (K0 smoothing stats, K1 psi,
K2 fused INT8 forward, K3 backward prep, K4 fused INT8 backward, K5 dQ finalize) over one
batch of the config's synthetic inputs, through the C ABI (libsage.so).
ops = 14 * B*H*N^2*d * f (f = 1/2 causal), FlashAttention convention.
Multi-GPU (torchrun, NCCL): each rank processes its own batch of the config (distinct
per-head seeds); no collective on the data path ("scaling": "weak"); the reported
time is the max over ranks.
"""
import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2603_02170_b200.inputs import CONFIGS, config_inputs  # noqa: E402

METRIC = "fwd+bwd attention TOPS vs INT8 peak at seqlen 1K–32K; rel-L2 of dQ/dK/dV"
DEFAULT_CONFIG = "C2"  # BASELINE.json configs[1], fits one GPU


def ops_of(c, batch=None):
    b = c.batch if batch is None else batch
    f = 0.5 if c.causal else 1.0
    return 14.0 * b * c.heads * c.seqlen ** 2 * c.head_dim * f


def bwd_kernel_ops(c):
    """K4 algorithmic ops per launch: S recompute, dV, dP, dQ, dK = 10 B H N^2 d f."""
    f = 0.5 if c.causal else 1.0
    return 10.0 * c.batch * c.heads * c.seqlen ** 2 * c.head_dim * f


def peaks():
    p = {}
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


def rank_head_offset(c, rank):
    """First global head index of this rank's batch: ranks own disjoint (batch x head) ranges
    (weak scaling, no data-path collective) and, with per-head seeds, a head's
    data does not depend on the world size."""
    return rank * c.batch * c.heads


def max_over_ranks(x, dist, device=None):
    """Max of a per-rank float over all ranks (the timing reduction; identity without dist)."""
    if dist is None:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


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


# ---------------------------------------------------------------------- CPU oracle (baseline / reference arm)
def oracle_sample(c, n_heads, seed_offset=0):
    """Time the oracle (as it stands) on n_heads heads of the config: fwd + bwd."""
    import numpy as np

    import oracle
    from paper_2603_02170_b200.inputs import make_inputs
    oracle.build()
    q, k, v, do = make_inputs(1, n_heads, c.seqlen, c.head_dim, c.recipe, seed=c.seed + seed_offset)
    cv = lambda t: t.float().numpy().astype(np.float64).reshape(n_heads, c.seqlen, c.head_dim)
    q, k, v, do = map(cv, (q, k, v, do))
    kw = dict(causal=c.causal, k_smooth=c.k_smooth, q_smooth=c.q_smooth)
    t0 = time.perf_counter()
    f = oracle.fwd(q, k, v, **kw)
    o_st = torch.from_numpy(f["o"]).to(torch.bfloat16).double().numpy()
    oracle.bwd(q, k, v, o_st, do, f["lse"], **kw)
    dt = time.perf_counter() - t0
    return dt, oracle.max_threads()


def cpu_baseline(c, budget_s=20.0):
    """Bounded sample: enough heads for ~budget_s of CPU work at the observed per-head rate."""
    cores = os.cpu_count() or 1
    n = max(1, min(c.batch * c.heads, cores))
    dt, threads = oracle_sample(c, n)
    ops = ops_of(c) / (c.batch * c.heads) * n
    sample = f"{n} heads of {c.name} (N={c.seqlen}, d={c.head_dim}) fwd+bwd, {threads} OpenMP threads"
    return {"value": ops / dt / 1e12, "unit": "TOPS", "cores": threads, "kind": "oracle", "sample": sample,
            "seconds": dt}


def run_reference(args, c, rank, world):
    """--impl reference: the CPU oracle on the host cores (the only other place bench runs oracle/)."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    n = max(1, min(c.batch * c.heads, cores))
    times = []
    for s in range(args.warmup + args.steps):
        dt, threads = oracle_sample(c, n, seed_offset=s)
        if s >= args.warmup:
            times.append(dt)
    ops = ops_of(c) / (c.batch * c.heads) * n
    tot = sum(times)
    value = ops * len(times) / tot / 1e12
    sample = f"{n} heads of {c.name} per step (N={c.seqlen}, d={c.head_dim}) fwd+bwd, {threads} OpenMP threads"
    line = {"metric": METRIC, "value": value, "unit": "TOPS", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i8/f64",
            "data": "synthetic", "config": config_dict(c, "n/a (CPU)"),
            "cpu_baseline": {"value": value, "unit": "TOPS", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(c, l2, qk_norm=False, p_u8=False, deterministic=False, fine_bwd=False):
    return {"workload": f"{c.name}: B={c.batch} H={c.heads} N={c.seqlen} d={c.head_dim} "
                        f"{'causal' if c.causal else 'non-causal'} K-smooth={c.k_smooth} Q-smooth={c.q_smooth} "
                        f"inputs={c.recipe}" + (" +QK-norm (fused)" if qk_norm else "") + (" P^ u8" if p_u8 else "")
                        + (" deterministic" if deterministic else "") + (" fine-bwd" if fine_bwd else ""),
            "batch": c.batch, "heads": c.heads, "seqlen": c.seqlen, "head_dim": c.head_dim, "causal": c.causal,
            "k_smooth": c.k_smooth, "q_smooth": c.q_smooth, "qk_norm": qk_norm, "p_u8": p_u8,
            "deterministic": deterministic, "fine_bwd": fine_bwd, "l2": l2}


# ---------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="sage", choices=["sage", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="head chunks of the pipelined e2e step (0: about 16 MB of inputs per chunk, at most 16)")
    ap.add_argument("--qk-norm", action="store_true",
                    help="QK-norm fused in front of the path (sage_fwd_qknorm / sage_bwd_qknorm, C5's ablation)")
    ap.add_argument("--p-u8", action="store_true", help="unsigned P^ variant (SAGE_P_U8)")
    ap.add_argument("--deterministic", action="store_true", help="bitwise reproducible dQ (SAGE_DETERMINISTIC)")
    ap.add_argument("--fine-bwd", action="store_true", help="per-key / per-query backward psi (SAGE_FINE_BWD)")
    args = ap.parse_args()
    assert args.warmup >= 3, "at least 3 warm-up steps"
    c = CONFIGS[args.config]
    dist, rank, world, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, c, rank, world)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    from paper_2603_02170_b200 import sage
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    # this rank's batch: distinct heads per rank (weak scaling), seeded on the CPU
    q, k, v, do = config_inputs(c, head_offset=rank_head_offset(c, rank))
    host = [t.pin_memory() for t in (q, k, v, do)]
    qd, kd, vd, dod = (t.to(dev) for t in host)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    kw = dict(causal=c.causal, k_smooth=c.k_smooth, q_smooth=c.q_smooth, p_u8=args.p_u8)
    if args.deterministic:
        kw["deterministic"] = True
    if args.fine_bwd:
        kw["fine_bwd"] = True
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
    value = ops_of(c) * world / (ms * 1e-3) / 1e12

    # e2e through the public API with host buffers: H2D of q, k, v, dO and D2H of o, dq, dk, dv every
    # step.  The heads are independent, so the step is pipelined over head chunks on
    # three streams: chunk k's H2D, chunk k-1's sage_fwd + sage_bwd and chunk k-2's D2H overlap (the
    # copies are full duplex).  The QK-norm variant's dgamma sums over all heads: serial there.
    outs_h = [torch.empty_like(h).pin_memory() for h in host]
    e2e_ms = []
    BH = c.batch * c.heads
    in_bytes = sum(h.numel() * h.element_size() for h in host)
    auto_chunks = max(1, min(16, in_bytes // (16 << 20)))  # measured: 8 at C2, 16 at C3
    n_chunks = 1 if (args.qk_norm or args.e2e_steps == 0) else min(args.e2e_chunks or auto_chunks, BH)
    bounds = [(BH * i // n_chunks, BH * (i + 1) // n_chunks) for i in range(n_chunks)]
    flat = lambda t: t.view(BH, c.seqlen, c.head_dim)
    chunk = lambda t, a, b: flat(t)[a:b].unsqueeze(0)  # [1, heads of the chunk, N, d], contiguous
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    if n_chunks > 1:
        ctxs = [sage.forward(chunk(qd, a, b), chunk(kd, a, b), chunk(vd, a, b), **kw)[2] for a, b in bounds]
    for s in range(args.e2e_steps + 1):
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
            for i, (lo, hi) in enumerate(bounds):
                with torch.cuda.stream(s_in):
                    for dst, src in zip((qd, kd, vd, dod), host):
                        chunk(dst, lo, hi).copy_(chunk(src, lo, hi), non_blocking=True)
                stream.wait_stream(s_in)
                qc, kc, vc, oc, doc, dqc, dkc, dvc = (chunk(t, lo, hi) for t in (qd, kd, vd, o, dod, dq, dk, dv))
                lc = lse.view(BH, c.seqlen)[lo:hi].unsqueeze(0)
                sage.forward(qc, kc, vc, out=oc, lse=lc, ctx=ctxs[i].buf, **kw)
                sage.backward(ctxs[i], vc, oc, lc, doc, dq=dqc, dk=dkc, dv=dvc)
                s_out.wait_stream(stream)
                with torch.cuda.stream(s_out):
                    for dst, src in zip(outs_h, (o, dq, dk, dv)):
                        chunk(dst, lo, hi).copy_(chunk(src, lo, hi), non_blocking=True)
        b_ev.record(s_out)
        torch.cuda.synchronize()
        if s > 0:
            e2e_ms.append(a_ev.elapsed_time(b_ev))
    te_ms = max_over_ranks(sum(e2e_ms) / max(1, len(e2e_ms)), dist, dev)
    nbytes = sum(h.numel() * h.element_size() for h in host)
    e2e = None
    if e2e_ms:
        e2e = {"value": ops_of(c) * world / (te_ms * 1e-3) / 1e12, "unit": "TOPS",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": te_ms,
               "pipeline": f"{n_chunks} head chunks, H2D / compute / D2H on three streams"}

    if rank == 0:
        pk = peaks()
        bwd_ms = prof["bwd_ms"] / max(1, prof["n_bwd"])
        fwd_ms = prof["fwd_ms"] / max(1, prof["n_fwd"])
        achieved = bwd_kernel_ops(c) / (bwd_ms * 1e-3) / 1e12
        traffic, traffic_src = traffic_from_profile(c.name)
        roof = {"bound": "tensor", "kernel": "sage_bwd_kernel (K4)", "achieved": achieved,
                "peak": pk["bwd_mixed"], "unit": "TFLOP/s", "frac": achieved / pk["bwd_mixed"],
                "traffic": traffic, "traffic_note": f"ncu dram__bytes_read+write.sum per launch, profiles/{traffic_src}"
                if traffic else None,
                "peak_note": f"{pk['src']} bf16 {pk['bf16']} TF/s x 5/3 (8/10 of K4's work INT8 at 2x bf16, 2/10 bf16)",
                "kernel_ms": bwd_ms, "share_of_step": bwd_ms / ms, "fwd_kernel_ms": fwd_ms,
                "fwd_share_of_step": fwd_ms / ms}
        line = {"metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "i8/bf16", "data": "synthetic",
                "config": config_dict(c, "flushed between timed steps (256 MiB write, untimed)", args.qk_norm,
                                      args.p_u8, args.deterministic, args.fine_bwd),
                "frac_of_int8_peak": value / world / pk["int8"], "int8_peak_tops": pk["int8"],
                "roofline": roof, "e2e": e2e, "gpu_launches": prof["launches"], "clocks": clk.summary()}
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(c)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
