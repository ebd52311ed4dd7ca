"""Build libbloch_b200.so in-tree with nvcc for sm_100a (no torch JIT cache).

``python -m paper_1305_6861_b200.build`` or ``build()`` from ``__graft_entry__``.
The shared library lands next to this file so it travels with the repo
snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_NAME = "libbloch_b200.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)

SOURCES = ["bloch_kernels.cu", "bloch_capi.cu", "program.cpp", "raster_kernels.cu", "contract_kernels.cu", "resident_kernels.cu"]
HEADERS = ["kernels.h", "program.h", "program_host.h", "raster.h", "contract.h", "resident.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the Bloch engine must be built with CUDA 12.9 nvcc")


def source_hash() -> str:
    """16 hex digits identifying the kernel sources (csrc/ + the C-ABI header).  nvcc's output is not
    bit-reproducible from one build to the next, so measurements that must be matched to a build (the ncu
    counters bench.py reads, profiles/ncu_counters.json) are keyed on this, not on the .so file."""
    import hashlib

    h = hashlib.sha256()
    for name in sorted(SOURCES + HEADERS):
        h.update(name.encode())
        with open(os.path.join(CSRC, name), "rb") as fh:
            h.update(fh.read())
    with open(os.path.join(ROOT, "include", "bloch_b200.h"), "rb") as fh:
        h.update(fh.read())
    return h.hexdigest()[:16]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile the library; ``out``/``defines`` build variants for A/B timing (tools/ab.sh)."""
    target = out or LIB_PATH
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "bloch_b200.h"),
        os.path.abspath(__file__),
    ]
    if not force and not defines and not _stale(target, deps):
        return target
    # one object per source, compiled in parallel and only when stale (A/B builds with defines: their own objects)
    import hashlib
    from concurrent.futures import ThreadPoolExecutor

    tag = hashlib.sha1(" ".join(defines).encode()).hexdigest()[:8] if defines else "base"
    objdir = os.path.join(CSRC, "_obj", tag)
    os.makedirs(objdir, exist_ok=True)
    hdrs = [d for d in deps if d not in srcs]
    common = [nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas",
              "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"), *[f"-D{d}" for d in defines]]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if force or _stale(obj, [src] + hdrs):
            cmd = [*common, "-c", src, "-o", obj]
            res = subprocess.run(cmd, capture_output=True, text=True)
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
            if verbose:
                sys.stderr.write(res.stdout + res.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(srcs)) as pool:
        objs = list(pool.map(compile_one, srcs))
    cmd = [nvcc_path(), *ARCH, "-shared", "-o", target + ".tmp", *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    # python -m paper_1305_6861_b200.build [--force] [-v] [--out PATH] [-DNAME=VALUE ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    print(build(force="--force" in args, verbose="-v" in args, out=out,
                defines=[a[2:] for a in args if a.startswith("-D")]))
