"""Build libsage.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsage.so")
TRACE_LIB = os.path.join(HERE, "libsage_trace.so")  # profiling build only
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

# -gencode arch=compute_100a,code=sm_100a: plain -arch=sm_100a embeds compute_100 PTX
# that rejects tcgen05.  No --use_fast_math (bit-exact quantiser, reading A4).
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-DSAGE_WAIT_HINT=" + os.environ.get("SAGE_WAIT_HINT", "0"),
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-shared",
         "-I" + os.path.join(HERE, "..", "include")]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(HERE, "..", "include", "sage.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def _link(lib, defines, verbose, tag=None):
    tag = tag or ("trace" if defines else "prod")
    objs = []
    for src in sources():
        obj = os.path.join(CSRC, "build", tag, os.path.basename(src) + ".o")
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        cmd = [NVCC] + [f for f in FLAGS if f != "-shared"] + defines + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-Xcompiler", "-fPIC", "-o", tmp] + objs + ["-lcudart"])
    os.replace(tmp, lib)


def build(force=False, verbose=False, trace=False):
    """Build libsage.so; with trace=True also libsage_trace.so (K4 timeline/ablation hooks)."""
    if force or _stale():
        _link(LIB, [], verbose)
    if trace:
        _link(TRACE_LIB, ["-DSAGE_TRACE=1"], verbose)
    return LIB


def build_variant(name, defines, verbose=False):
    """Profiling only: libsage_<name>.so built with extra -D flags (selected with SAGE_LIB=...)."""
    lib = os.path.join(HERE, f"libsage_{name}.so")
    _link(lib, list(defines), verbose, tag=name)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv)
    print(LIB)
