"""Build the sm_100a shared library ``_lib/libqfswe.so`` in-tree.

    python -m paper_1904_08684_b200.build

Regenerates the literal-constant headers (``codegen.py``) and compiles
``csrc/qf_kernels.cu`` with nvcc for ``compute_100a``/``sm_100a`` only.
The result is a plain C-ABI library (include/qfswe.h); no torch types cross
the boundary.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libqfswe.so"
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2", "-shared",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + \
        sorted((CSRC / "generated").glob("*.cuh")) + [ROOT / "include" / "qfswe.h"]


def _digest() -> str:
    h = hashlib.sha256()
    for p in _sources():
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS + os.environ.get("QF_NVCC_EXTRA", "").split()).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    from .codegen import generate

    generate()
    LIB_DIR.mkdir(exist_ok=True)
    stamp = LIB_DIR / "libqfswe.sha256"
    dig = _digest()
    if not force and LIB.exists() and stamp.exists() and stamp.read_text() == dig:
        return LIB
    extra = os.environ.get("QF_NVCC_EXTRA", "").split()
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", str(LIB), str(CSRC / "qf_kernels.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stderr}")
    if verbose:
        print(res.stderr)
    stamp.write_text(dig)
    return LIB


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
