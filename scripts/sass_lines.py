"""Static SASS instruction histogram per source-line range of one kernel (fully unrolled loops ->
static count ~ per-tile dynamic count).  usage: sass_lines.py file.cu kernel_substr L0-L1[,L0-L1...] [flags]"""
import re, subprocess, sys, collections, os
src, ksub, ranges = sys.argv[1], sys.argv[2], sys.argv[3]
flags = sys.argv[4:]
cub = "/tmp/_sl.cubin"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                       "-lineinfo", "-DSAGE_WAIT_HINT=0", "-cubin", "-o", cub, src] + flags)
out = subprocess.check_output(["/usr/local/cuda/bin/nvdisasm", "-g", cub], text=True)
rs = [tuple(map(int, r.split("-"))) for r in ranges.split(",")]
fn = None; ln = 0; base = os.path.basename(src)
hist = {r: collections.Counter() for r in rs}
for line in out.splitlines():
    if line.startswith(".text."):
        fn = line
        continue
    m = re.search(r'line (\d+)', line)
    if m and base in line:
        ln = int(m.group(1))
        continue
    if fn is None or ksub not in fn:
        continue
    m = re.match(r'\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)', line)
    if not m:
        continue
    op = m.group(2).split(".")[0]
    for r in rs:
        if r[0] <= ln <= r[1]:
            hist[r][op] += 1
for r in rs:
    h = hist[r]
    print(f"lines {r[0]}-{r[1]}: total {sum(h.values())}")
    print("   " + "  ".join(f"{k}:{v}" for k, v in h.most_common(30)))
