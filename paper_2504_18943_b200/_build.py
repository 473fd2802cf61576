"""Builds the CUDA engine in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The shared library lands in ``paper_2504_18943_b200/_lib/`` so that it travels with the
repository snapshot to the GPU box.  ``__graft_entry__.build()`` calls ``build_native``.

The enumeration kernels are templates over (lane width, operator); ``csrc/inst.cu`` is compiled
once per (lane width, narrow | wide) beside ``csrc/engine.cu`` (host side, finalisation and
exchange kernels), all objects in parallel, then linked into one library.
"""

from __future__ import annotations

import concurrent.futures
import os
import pathlib
import shutil
import subprocess

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
OBJ_DIR = LIB_DIR / "obj"
LIB_PATH = LIB_DIR / "libltlsynth_b200.so"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = [*ARCH_FLAGS, "-Xfatbin", "-compress-all", "-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2,-Wall"]
LINK_FLAGS = [*ARCH_FLAGS, "-shared", "-cudart", "static"]
LANE_WIDTHS = (8, 16, 32, 64)


def _units() -> list[tuple[str, str, list[str]]]:
    """(object name, source file, extra defines) of every translation unit."""
    units = [("engine", "engine.cu", [])]
    for lw in LANE_WIDTHS:
        units.append((f"narrow_lw{lw}", "inst.cu", [f"-DLTLB200_INST_LW={lw}", "-DLTLB200_INST_WIDE=0"]))
        units.append((f"wide_lw{lw}", "inst.cu", [f"-DLTLB200_INST_LW={lw}", "-DLTLB200_INST_WIDE=1"]))
    units.append(("wide_regex", "inst.cu", ["-DLTLB200_INST_LW=1", "-DLTLB200_INST_WIDE=1"]))  # regex grammar (wide2_regex.cuh)
    return units


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA engine cannot be built")


def _newest_source() -> float:
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [PKG.parent / "include" / "ltlsynth_b200.h"]
    return max(p.stat().st_mtime for p in deps)


def _stale(path: pathlib.Path) -> bool:
    return not path.exists() or path.stat().st_mtime < _newest_source()


def build_native(force: bool = False, verbose: bool = False, defines=(), out: pathlib.Path | None = None) -> pathlib.Path:
    """``defines``/``out`` build a tuning variant (e.g. ("LTLB200_PROBE_BATCH=2",)) beside the default library."""
    target = pathlib.Path(out) if out else LIB_PATH
    variant = out is not None or bool(defines)
    if not force and not variant and not _stale(LIB_PATH):
        return LIB_PATH
    obj_dir = OBJ_DIR if not variant else LIB_DIR / ("obj_" + target.stem)
    obj_dir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    extra = [*(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines]]

    def compile_unit(unit):
        name, source, unit_defines = unit
        obj = obj_dir / f"{name}.o"
        if not force and not variant and not _stale(obj):
            return obj, ""
        cmd = [nvcc, *COMPILE_FLAGS, *extra, *unit_defines, "-c", "-o", str(obj), str(CSRC / source)]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed on {name}:\n" + proc.stdout + proc.stderr)
        return obj, proc.stdout + proc.stderr

    with concurrent.futures.ThreadPoolExecutor(max_workers=min(len(_units()), os.cpu_count() or 4)) as pool:
        results = list(pool.map(compile_unit, _units()))
    if verbose:
        for obj, log in results:
            print(f"---- {obj.name}\n{log}")
    proc = subprocess.run([nvcc, *LINK_FLAGS, "-o", str(target), *[str(obj) for obj, _ in results]], capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("link failed:\n" + proc.stdout + proc.stderr)
    return target


def build_tools() -> None:
    """Measurement tools (not part of the product path): the random-probe ceiling microbenchmark
    that bench.py runs beside the kernel."""
    root = PKG.parent / "tools"
    for name in ("random_probe_bench", "window_probe_bench"):
        src, exe = root / f"{name}.cu", root / name
        if exe.exists() and exe.stat().st_mtime >= src.stat().st_mtime:
            continue
        proc = subprocess.run([_nvcc(), *ARCH_FLAGS, "-O3", "-o", str(exe), str(src)], capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + proc.stdout + proc.stderr)


if __name__ == "__main__":
    import sys

    print(build_native(force=True, verbose="-v" in sys.argv))
