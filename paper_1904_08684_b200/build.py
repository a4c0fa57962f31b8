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


def compile_user_module(source: str) -> bytes:
    """nvcc a user-scenario module (scenario.user_device_source) to an sm_100a
    cubin; cached per source digest in the temp directory."""
    import tempfile

    flags = ["-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
             "--expt-relaxed-constexpr", "-I", str(CSRC)]
    dig = hashlib.sha256((source + " ".join(flags)).encode())
    for p in sorted(CSRC.glob("*.cuh")) + sorted((CSRC / "generated").glob("*.cuh")):
        dig.update(p.read_bytes())
    cache = Path(tempfile.gettempdir()) / "qfswe_user"
    cache.mkdir(exist_ok=True)
    out = cache / f"{dig.hexdigest()[:32]}.cubin"
    if not out.exists():
        src = cache / f"{dig.hexdigest()[:32]}.cu"
        src.write_text(source)
        tmp = out.with_suffix(f".{os.getpid()}.tmp")
        res = subprocess.run([nvcc(), *flags, "-o", str(tmp), str(src)], capture_output=True,
                             text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc (user scenario module) failed:\n{res.stderr[-4000:]}")
        os.replace(tmp, out)
    return out.read_bytes()


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
