"""In-tree build of the native libraries (no JIT cache, no pip install).

* ``_lib/libsnplan.so``  -- C++17 planner (schedule, liveness, offload, recompute,
  block pool, LRU cache, event tape).  Host only, built with g++.
* ``_lib/libsnexec.so``  -- CUDA executor + sm_100a kernels, built with nvcc
  ``-gencode arch=compute_100a,code=sm_100a``; links libsnplan.so.
* ``_lib/libsntest.so``  -- test-only hooks and hardware probes (``csrc/testing``:
  kernel-level parity entry points, tcgen05 rate / layout probes); links
  libsnexec.so and is never loaded by the training path.

Both are plain C-ABI libraries loaded with ctypes (see ``_native.py``); the
declarations live in ``include/superneurons.h``.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "_lib"
REPO = PKG.parent
INCLUDE = REPO / "include"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

# The planner's float arithmetic must follow the reference's IEEE-double
# operation order exactly: no contraction into FMA, no fast-math.
PLAN_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
              "-Wall", "-Wextra", "-Wno-unused-parameter"]


def _sources(sub: str, exts: tuple[str, ...]) -> list[Path]:
    root = CSRC / sub
    return sorted(p for p in root.rglob("*") if p.suffix in exts)


def _digest(paths: list[Path], extra: list[str]) -> str:
    h = hashlib.sha256()
    for p in paths:
        h.update(str(p).encode())
        h.update(p.read_bytes())
    h.update(" ".join(extra).encode())
    return h.hexdigest()


def _up_to_date(out: Path, digest: str) -> bool:
    stamp = out.with_suffix(out.suffix + ".sha")
    return out.exists() and stamp.exists() and stamp.read_text() == digest


def _stamp(out: Path, digest: str) -> None:
    out.with_suffix(out.suffix + ".sha").write_text(digest)


def _run(cmd: list[str]) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")


def build_planner(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libsnplan.so"
    srcs = _sources("planner", (".cpp",))
    headers = _sources("planner", (".hpp", ".h")) + sorted(INCLUDE.glob("*.h"))
    digest = _digest(srcs + headers, PLAN_FLAGS)
    if not force and _up_to_date(out, digest):
        return out
    cmd = ["g++", *PLAN_FLAGS, "-shared", f"-I{INCLUDE}", f"-I{CSRC}",
           *map(str, srcs), "-o", str(out)]
    _run(cmd)
    _stamp(out, digest)
    return out


def build_exec(force: bool = False) -> Path:
    plan = build_planner(force)
    out = LIB / "libsnexec.so"
    srcs = _sources("exec", (".cu", ".cpp")) + _sources("kernels", (".cu",))
    headers = (_sources("exec", (".cuh", ".hpp", ".h")) + _sources("kernels", (".cuh", ".h", ".hpp"))
               + _sources("planner", (".hpp",)) + sorted(INCLUDE.glob("*.h")))
    flags = ["-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
             "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr"]
    digest = _digest(srcs + headers + [plan], flags)
    if not force and _up_to_date(out, digest):
        return out
    objdir = LIB / "obj"
    objdir.mkdir(exist_ok=True)
    objs = [str(objdir / (src.stem + ".o")) for src in srcs]
    import concurrent.futures as cf
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as pool:
        list(pool.map(lambda so: _run([NVCC, *flags, f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(so[0]), "-o", so[1]]),
                      zip(srcs, objs)))
    _run([NVCC, *ARCH, "-shared", *objs, "-o", str(out), f"-L{LIB}", "-lsnplan", "-ldl",
          "-Xlinker", "-rpath,$ORIGIN"])
    _stamp(out, digest)
    return out


def build_testing(force: bool = False) -> Path:
    exe = build_exec(force)
    out = LIB / "libsntest.so"
    srcs = _sources("testing", (".cu",))
    headers = _sources("kernels", (".cuh", ".h", ".hpp")) + sorted(INCLUDE.glob("*.h"))
    flags = ["-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
    digest = _digest(srcs + headers + [exe], flags)
    if not force and _up_to_date(out, digest):
        return out
    objdir = LIB / "obj"
    objdir.mkdir(exist_ok=True)
    objs = [str(objdir / ("test_" + src.stem + ".o")) for src in srcs]
    import concurrent.futures as cf
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as pool:
        list(pool.map(lambda so: _run([NVCC, *flags, f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(so[0]), "-o", so[1]]),
                      zip(srcs, objs)))
    _run([NVCC, *ARCH, "-shared", *objs, "-o", str(out), f"-L{LIB}", "-lsnexec", "-lsnplan",
          "-Xlinker", "-rpath,$ORIGIN"])
    _stamp(out, digest)
    return out


def build_all(force: bool = False) -> None:
    build_planner(force)
    build_exec(force)
    build_testing(force)


if __name__ == "__main__":
    import sys
    build_all(force="--force" in sys.argv)
    print("built", *(p.name for p in LIB.glob("*.so")))
