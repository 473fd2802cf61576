#!/usr/bin/env python3
"""Installs the UNMODIFIED reference (`ltlsynth` 0.1.0, pure Python + numpy) into ``oracle/_ref/``.

    python oracle/build_ref.py

Build container only: ``/root/reference`` does not exist on the GPU box, ``oracle/_ref/`` travels there with the
repository snapshot (git-ignored, not gpurun-ignored).  ``bench.py --impl reference`` and its ``cpu_baseline`` leg
time this package -- the reference's own CPU implementation of the enumeration path -- beside the CUDA engine;
nothing in ``paper_2504_18943_b200`` imports it.  The reference is installed with pip from a scratch copy of its
source tree (its build writes ``*.egg-info`` next to ``pyproject.toml`` and ``/root/reference`` is read-only);
no reference source is copied into the tracked part of this repository.
"""

from __future__ import annotations

import pathlib
import shutil
import subprocess
import sys
import tempfile

HERE = pathlib.Path(__file__).resolve().parent
REFERENCE_PKG = pathlib.Path("/root/reference/pkg")
TARGET = HERE / "_ref"


def build_ref(force: bool = False) -> pathlib.Path | None:
    """None when the reference is not available here (the GPU box): whatever ``oracle/_ref`` holds is used as is."""
    if not (REFERENCE_PKG / "pyproject.toml").exists():
        return TARGET if (TARGET / "ltlsynth").exists() else None
    if (TARGET / "ltlsynth" / "engine.py").exists() and not force:
        return TARGET
    with tempfile.TemporaryDirectory() as tmp:
        scratch = pathlib.Path(tmp) / "pkg"
        shutil.copytree(REFERENCE_PKG, scratch)
        shutil.rmtree(TARGET, ignore_errors=True)
        subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index", "--no-build-isolation", "--no-deps",
                        "--target", str(TARGET), str(scratch)], check=True)
    return TARGET


if __name__ == "__main__":
    print(build_ref(force=True))
