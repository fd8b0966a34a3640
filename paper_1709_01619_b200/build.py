"""Build libhom2d.so in-tree with nvcc for sm_100a (B200).

    python -m paper_1709_01619_b200.build [--force]

Cross-compiles without a GPU.  The .so lands next to this file so that it
travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhom2d.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_dir() -> str:
    """The NCCL torch ships (nvidia-nccl wheel): linking it (with an rpath) makes
    the library and torch share one libnccl.so.2 whatever the import order."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.nccl (torch's NCCL) not found")
    return list(spec.submodule_search_locations)[0]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared",
         "-Xptxas", "-warn-spills"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "hom2d.h")]


def src_hash() -> str:
    import hashlib
    h = hashlib.sha256()
    for p in sorted(deps()):
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def stale() -> bool:
    """Content-based: the library is stale when the sources hash differs from the
    one recorded at build time (robust to snapshot copies that reset mtimes)."""
    if not os.path.exists(LIB) or not os.path.exists(LIB + ".srchash"):
        return True
    with open(LIB + ".srchash") as f:
        return f.read().strip() != src_hash()


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra=()) -> str:
    """Compile all csrc/*.cu into `out` (variants for A/B timing: out + extra -D flags)."""
    if out == LIB and not force and not stale():
        return LIB
    nd = nccl_dir()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include")]
    # one nvcc per translation unit, in parallel; then one link
    import concurrent.futures
    import tempfile
    tmp = tempfile.mkdtemp(prefix="hom2d_build_")
    objs = [os.path.join(tmp, os.path.basename(src) + ".o") for src in sources()]
    cflags = [f for f in FLAGS if f != "-shared"]
    cmds = []
    for src, obj in zip(sources(), objs):
        c = [NVCC, *ARCH, *cflags, *extra, *inc, "-c", "-o", obj, src]
        if verbose:
            c.insert(1, "-Xptxas=-v")
        cmds.append(c)
    with concurrent.futures.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for c in ex.map(lambda c: (subprocess.check_call(c), c)[1], cmds):
            if verbose:
                print(" ".join(c), flush=True)
    link = [NVCC, *ARCH, "-shared", "-o", out, *objs, "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
    subprocess.check_call(link)
    for o in objs:
        os.remove(o)
    os.rmdir(tmp)
    if out == LIB:
        with open(LIB + ".srchash", "w") as f:
            f.write(src_hash())
    return out


if __name__ == "__main__":
    # python -m paper_1709_01619_b200.build [--force] [-v] [--out PATH -DNAME=VAL ...]
    args = sys.argv[1:]
    out = LIB
    if "--out" in args:
        out = os.path.abspath(args[args.index("--out") + 1])
    extra = [a for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, out=out, extra=extra))
