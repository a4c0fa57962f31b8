"""Diagnostic: build compile-time knob variants of libqfswe.so (here, CPU)
and time them on the GPU (``run``), one subprocess per variant.

    python tools/variants.py build base= vsplit4=-DQF_VSPLIT=4 occ2=-DQF_OCC4=2
    python tools/variants.py run "3 4" 256            # on the GPU box
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
VAR = ROOT / "paper_1904_08684_b200" / "_lib" / "var"


def build(specs):
    from paper_1904_08684_b200 import build as B
    from paper_1904_08684_b200.codegen import generate

    generate()
    VAR.mkdir(parents=True, exist_ok=True)
    for spec in specs:
        name, _, flags = spec.partition("=")
        out = VAR / f"{name}.so"
        cmd = [B.nvcc(), *B.NVCC_FLAGS, *flags.split(), "-o", str(out), str(B.CSRC / "qf_kernels.cu")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        print(name, "ok" if r.returncode == 0 else r.stderr[-2000:])


def run(orders, n, scen, rounds=int(os.environ.get("QF_ROUNDS", "1"))):
    """Variants interleaved ``rounds`` times (box-to-box and drift noise is
    ~4 %, so compare within one call)."""
    for so in [so for _ in range(rounds) for so in sorted(VAR.glob("*.so"))]:
        env = dict(os.environ, QF_LIB=str(so))
        code = (f"import sys; sys.path.insert(0, {str(ROOT)!r}); from tools.order_timing import main; "
                f"main({n}, orders=({orders},), scen={scen!r})")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        out = r.stdout.strip().replace("\n", "\n    ")
        print(f"[{so.stem}]\n    {out or r.stderr[-800:]}", flush=True)


def execute(cmd):
    """Run a shell command once per variant with QF_LIB pointing at it."""
    for so in sorted(VAR.glob("*.so")):
        r = subprocess.run(cmd, shell=True, env=dict(os.environ, QF_LIB=str(so)),
                           capture_output=True, text=True, cwd=ROOT)
        out = (r.stdout.strip() or r.stderr[-800:]).replace("\n", "\n    ")
        print(f"[{so.stem}]\n    {out}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    elif sys.argv[1] == "exec":
        execute(" ".join(sys.argv[2:]))
    else:
        run(",".join(sys.argv[2].split()) if len(sys.argv) > 2 else "3,4",
            int(sys.argv[3]) if len(sys.argv) > 3 else 256,
            sys.argv[4] if len(sys.argv) > 4 else "bumps")
