"""p = 4 manufactured-solution errors from the CPU oracle (test fixture).

The reference has no p = 4 basis (symbolic.py:455-456), so the p = 4
convergence test compares the GPU errors with the oracle's p = 4 extension
(oracle/qfswe_oracle.py, exact Gram-Schmidt completion) on the overlapping
meshes.  Fields: the BASELINE MMS (U = H u, V = H v, xi mass source) over a
LINEAR bathymetry h_b = 1 + 0.1 x + 0.05 y (its P1 projection is exact, so
the design order k + 1 = 5 is reachable) and over the BASELINE bilinear
h_b = 1 + 0.1 x y.  SSP-RK3, dt = 2e-5, 1000 steps (t_end = 0.02, the C2
schedule), unit-square SW-NE meshes N = 4, 8.

    python tests/golden/make_sweep_p4.py      # writes sweep_p4_oracle.npz
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

HB = {"linear": "1 + x/10 + y/20", "bilinear": "1 + x*y/10"}
NS, DT, STEPS, K = (4, 8), 2e-5, 1000, 4


def mms(hb, **kw):
    from oracle import qfswe_oracle as O

    xi = "sin(2*pi*(x+y-t))/100"
    H = f"({hb} + {xi})"
    return O.sympy_scenario(xi, f"{H}*cos(2*pi*(x-t))/10", f"{H}*sin(2*pi*(y-t))/10", hb,
                            with_mass_source=True, **kw)


def main():
    from oracle import qfswe_oracle as O
    from paper_1904_08684_b200 import mesh as M

    out = {"n": np.array(NS), "dt": DT, "steps": STEPS}
    for name, hb in HB.items():
        errs = []
        for n in NS:
            t0 = time.time()
            m = M.build_unit_square_mesh(n)
            orc = O.OracleSolver(O.OMesh(m.vertices, m.triangles), mms(hb, dt=DT), K)
            c, _ = orc.project_initial()
            c, _, t = orc.run(c, 0.0, STEPS)
            errs.append(orc.l2_error(c, t))
            print(f"{name} N={n}: {errs[-1]} ({time.time() - t0:.0f} s)", flush=True)
        out[f"err_{name}"] = np.array(errs)
    np.savez_compressed(HERE / "sweep_p4_oracle.npz", **out)


if __name__ == "__main__":
    main()
