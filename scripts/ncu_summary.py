"""Summarise ncu reports / launch lists for profiles/ (run here, no GPU needed).

  python scripts/ncu_summary.py rep  <file.ncu-rep> [...]   key raw metrics + SASS op mix per kernel
  python scripts/ncu_summary.py launches <launches.csv>       per-kernel launch count, mean time, share
  python scripts/ncu_summary.py json <out.json> <prof_<tag>_<cfg>_<kernel>.ncu-rep> [...]
                                                             merge key counters per (kernel, config) into a JSON
                                                             file that bench.py reads for roofline.traffic
"""
import json
import os
import re
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sass__inst_executed_local_loads", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg"]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args + ["--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def rep(path):
    rows = ncu_csv(["-i", path, "--page", "raw"])
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print(f"### {vals[hdr.index('Kernel Name')][:110]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:82s} {vals[i]:>16s} {units[i]}")
    src = ncu_csv(["-i", path, "--page", "source", "--print-source=sass"])
    hdr = src[1]
    si, ie = hdr.index("Source"), hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    ops, stall, tot, tst = Counter(), Counter(), 0, 0
    for r in src[2:]:
        try:
            n, s = int(r[ie]), int(r[st])
        except (ValueError, IndexError):
            continue
        toks = r[si].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
        ops[op] += n
        stall[op] += s
        tot += n
        tst += s
    print(f"  SASS warp-instructions executed: {tot}")
    for op, n in ops.most_common(16):
        print(f"    {op:10s} {100 * n / tot:5.1f}% of inst   {100 * stall[op] / max(1, tst):5.1f}% of stall samples")


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[h + 1:]:
        agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    print(f"{'launches':>8s} {'mean us':>10s} {'share':>7s}  kernel   (cold-cache, serialised ncu launch list)")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {100 * sum(v) / total:6.1f}%  {k}")


def to_json(out, files):
    data = json.load(open(out)) if os.path.exists(out) else {"kernels": {}}
    for path in files:
        m = re.search(r"prof_([^_]+)_(C\d)_([a-z0-9_]+?)(?:_kernel)?\.ncu-rep$", os.path.basename(path))
        if not m:
            continue
        tag, cfg, kern = m.groups()
        rows = ncu_csv(["-i", path, "--page", "raw"])
        hdr, vals = rows[0], rows[2]
        get = lambda k: float(vals[hdr.index(k)].replace(",", "")) if k in hdr else None
        rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
        # ncu reports bytes with unit scaling in the units row (Kbyte/Mbyte/Gbyte)
        units = rows[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
        wr *= scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
        tscale = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
        t = get("gpu__time_duration.sum") * tscale.get(units[hdr.index("gpu__time_duration.sum")], 1e-9)
        data["kernels"].setdefault(kern, {})[cfg] = {
            "tag": tag, "report": os.path.basename(path), "time_s": t, "dram_read_bytes": rd,
            "dram_write_bytes": wr, "dram_bytes": rd + wr,
            "imma_pct": get("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active"),
            "hmma_pct": get("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active"),
            "xu_pct": get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "alu_pct": get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma_pct": get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "dram_pct": get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "warp_inst": get("smsp__inst_executed.sum")}
    json.dump(data, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(data, indent=1, sort_keys=True))


if __name__ == "__main__":
    mode, files = sys.argv[1], sys.argv[2:]
    if mode == "json":
        to_json(files[0], files[1:])
        sys.exit(0)
    for f in files:
        print(f"==== {f}")
        (rep if mode == "rep" else launches)(f)
