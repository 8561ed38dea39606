"""Build libsage.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo).

Translation units compile in parallel (one nvcc per source, both libraries at once); an object is
rebuilt when its source, any header or this file is newer than it.  ptxas -v output is kept per
object and summarised in csrc/build/<tag>/ptxas_spills.txt: every kernel instantiation that spills
registers to local memory is listed (a spill in a fused kernel is a performance regression to
explain).
"""
import glob
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsage.so")
TRACE_LIB = os.path.join(HERE, "libsage_trace.so")  # test / profiling build (tile dumps, timelines)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

# -gencode arch=compute_100a,code=sm_100a: plain -arch=sm_100a embeds compute_100 PTX
# that rejects tcgen05.  No --use_fast_math (bit-exact quantiser, reading A4).
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-DSAGE_WAIT_HINT=" + os.environ.get("SAGE_WAIT_HINT", "0"),
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v",
         "-diag-suppress", "177",
         "-I" + os.path.join(HERE, "..", "include")]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(HERE, "..", "include", "sage.h"), __file__]


def _newest_dep(src):
    return max(os.path.getmtime(p) for p in [src] + _headers())


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(_newest_dep(s) > t for s in sources())


def _obj(tag, src):
    return os.path.join(CSRC, "build", tag, os.path.basename(src) + ".o")


def _compile(src, obj, defines, verbose, force):
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= _newest_dep(src) and \
            os.path.exists(obj + ".ptxas"):
        return obj
    os.makedirs(os.path.dirname(obj), exist_ok=True)
    cmd = [NVCC] + FLAGS + defines + ["-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise subprocess.CalledProcessError(p.returncode, cmd)
    with open(obj + ".ptxas", "w") as f:
        f.write(p.stderr)
    return obj


_ENTRY = re.compile(r"Compiling entry function '(\S+)'")
_SPILL = re.compile(r"(\d+) bytes spill stores, (\d+) bytes spill loads")


def spills(objs):
    """[(kernel, store bytes, load bytes)] for every entry function that spills."""
    out = []
    for o in objs:
        cur = None
        for line in open(o + ".ptxas"):
            m = _ENTRY.search(line)
            if m:
                cur = m.group(1)
                continue
            m = _SPILL.search(line)
            if m and cur and (int(m.group(1)) or int(m.group(2))):
                out.append((cur, int(m.group(1)), int(m.group(2))))
    return out


def _demangle(names):
    try:
        p = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
        return p.stdout.splitlines()
    except OSError:
        return names


def _link(lib, objs):
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-Xcompiler", "-fPIC", "-o", tmp] + objs + ["-lcudart"])
    os.replace(tmp, lib)
    sp = spills(objs)
    names = _demangle([k for k, _, _ in sp])
    rep = os.path.join(os.path.dirname(objs[0]), "ptxas_spills.txt")
    with open(rep, "w") as f:
        for (k, st, ld), n in zip(sp, names):
            f.write(f"{st:5d} B stores {ld:5d} B loads  {n}\n")
    return sp


def _build_libs(jobs, verbose, force):
    """jobs: [(lib path, defines, tag)] -> compile every object of every lib in parallel, then link."""
    tasks = [(lib, src, _obj(tag, src), defines) for lib, defines, tag in jobs for src in sources()]
    with ThreadPoolExecutor(max_workers=min(len(tasks), os.cpu_count() or 4)) as ex:
        list(ex.map(lambda t: _compile(t[1], t[2], t[3], verbose, force), tasks))
    for lib, defines, tag in jobs:
        _link(lib, [_obj(tag, s) for s in sources()])


def build(force=False, verbose=False, trace=False):
    """Build libsage.so; with trace=True also libsage_trace.so (test-only tile dumps, timelines)."""
    jobs = []
    if force or _stale():
        jobs.append((LIB, [], "prod"))
    if trace and (force or not os.path.exists(TRACE_LIB) or
                  any(_newest_dep(s) > os.path.getmtime(TRACE_LIB) for s in sources())):
        jobs.append((TRACE_LIB, ["-DSAGE_TRACE=1"], "trace"))
    if jobs:
        _build_libs(jobs, verbose, force)
    return LIB


def build_variant(name, defines, verbose=False):
    """Profiling only: libsage_<name>.so built with extra -D flags (selected with SAGE_LIB=...)."""
    lib = os.path.join(HERE, f"libsage_{name}.so")
    _build_libs([(lib, list(defines), name)], verbose, False)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv)
    rep = os.path.join(CSRC, "build", "prod", "ptxas_spills.txt")
    if os.path.exists(rep):
        print(open(rep).read(), end="")
    print(LIB)
