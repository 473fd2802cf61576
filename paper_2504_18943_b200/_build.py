"""Builds the CUDA engine in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The shared library lands in ``paper_2504_18943_b200/_lib/`` so that it travels with the
repository snapshot to the GPU box.  ``__graft_entry__.build()`` calls ``build_native``.
"""

from __future__ import annotations

import os
import pathlib
import shutil
import subprocess

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB_PATH = LIB_DIR / "libltlsynth_b200.so"

SOURCES = ["engine.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2,-Wall",
    "-shared", "-cudart", "static",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA engine cannot be built")


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "ltlsynth_b200.h"]
    return any(p.stat().st_mtime > built for p in deps)


def build_native(force: bool = False, verbose: bool = False, defines=(), out: pathlib.Path | None = None) -> pathlib.Path:
    """``defines``/``out`` build a tuning variant (e.g. ("LTLB200_PROBE_BATCH=2",)) beside the default library."""
    target = pathlib.Path(out) if out else LIB_PATH
    if not force and out is None and not _stale():
        return LIB_PATH
    LIB_DIR.mkdir(exist_ok=True)
    cmd = [_nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines],
           "-o", str(target), *[str(CSRC / s) for s in SOURCES]]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + proc.stdout + proc.stderr)
    if verbose:
        print(proc.stdout + proc.stderr)
    return target


def build_tools() -> None:
    """Measurement tools (not part of the product path): the random-probe ceiling microbenchmark
    that bench.py runs beside the kernel."""
    root = PKG.parent / "tools"
    for name in ("random_probe_bench", "window_probe_bench"):
        src, exe = root / f"{name}.cu", root / name
        if exe.exists() and exe.stat().st_mtime >= src.stat().st_mtime:
            continue
        proc = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", str(exe), str(src)],
                              capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + proc.stdout + proc.stderr)


if __name__ == "__main__":
    import sys

    print(build_native(force=True, verbose="-v" in sys.argv))
