"""Build libndf_b200.so in-tree: nvcc for sm_100a, one object per .cu, then link.

    python -m paper_2307_02203_b200.build [--verbose] [--ptxas-info]

The shared library is written next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
BUILD = os.path.join(os.path.dirname(HERE), "build", "obj")
LIB = os.path.join(HERE, "libndf_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", INCLUDE, "-I", CSRC]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found; cannot build libndf_b200")
    return path


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _sha(*parts) -> str:
    h = hashlib.sha256()
    for p in parts:
        h.update(p if isinstance(p, bytes) else str(p).encode())
    return h.hexdigest()


def _file_sha(path) -> str:
    with open(path, "rb") as fh:
        return _sha(fh.read())


def _compile(src, verbose=False, ptxas_info=False):
    """Compile one .cu unless its object is current.  Staleness is keyed on a hash of
    the source, every header it may include and the flags -- not on mtimes -- so a
    copied, restored or half-written object is never mistaken for current."""
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    deps = [src] + sorted(os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith(".cuh"))
    deps.append(os.path.join(INCLUDE, "ndf_b200.h"))
    key = _sha(*[_file_sha(d) for d in deps], *ARCH, *FLAGS)
    stamp = obj + ".sha"
    if (not ptxas_info and os.path.exists(obj) and os.path.exists(stamp)
            and open(stamp).read() == key + _file_sha(obj)):
        return obj, ""
    cmd = [nvcc(), *ARCH, *FLAGS, "-c", src, "-o", obj]
    if ptxas_info:
        cmd.insert(1, "-Xptxas=-v")
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
    with open(stamp, "w") as fh:
        fh.write(key + _file_sha(obj))
    return obj, res.stderr


def build(verbose=False, ptxas_info=False, force=False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose, ptxas_info or force), srcs))
    objs = [o for o, _ in results]
    if ptxas_info:
        for (o, log) in results:
            print(f"== {os.path.basename(o)}\n{log}")
    # relink unless the library is byte-for-byte the one linked from these objects
    key = _sha(*[_file_sha(o) for o in objs])
    stamp = os.path.join(BUILD, "libndf_b200.sha")
    current = (os.path.exists(LIB) and os.path.exists(stamp)
               and open(stamp).read() == key + _file_sha(LIB))
    if force or not current:
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
        with open(stamp, "w") as fh:
            fh.write(key + _file_sha(LIB))
    return LIB


if __name__ == "__main__":
    lib = build(verbose="--verbose" in sys.argv, ptxas_info="--ptxas-info" in sys.argv,
                force="--force" in sys.argv)
    print(lib)
