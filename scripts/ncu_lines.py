"""Per-source-line hot spots of an ncu report (run here): stall samples and warp-instructions.

  python scripts/ncu_lines.py <rep.ncu-rep> [top]
Uses the cuda,sass source page (needs -lineinfo); one row per CUDA source line.
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, hdr, fname = [], None, None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or r[2] != "-":   # keep the per-CUDA-line aggregate rows
        continue
    try:
        s, n = float(r[4] or 0), float(r[7] or 0)
    except ValueError:
        continue
    stalls = {}
    for k, v in zip(hdr, r):
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                if float(v):
                    stalls[k[6:]] = float(v)
            except ValueError:
                pass
    if s or n:
        rows.append((s, n, fname, r[0], r[1].strip()[:68], stalls))
tot_s = sum(r[0] for r in rows) or 1
tot_n = sum(r[1] for r in rows) or 1
print(f"total stall samples {tot_s:.0f}, warp-instructions {tot_n:.0f}")
for s, n, f, ln, src, st in sorted(rows, key=lambda r: -r[0])[:top]:
    big = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100*s/tot_s:5.1f}% smp {100*n/tot_n:5.1f}% ins {f[:10]}:{ln:>4} {src:68s} {' '.join(f'{k}={100*v/tot_s:.1f}' for k,v in big)}")
