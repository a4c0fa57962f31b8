"""Drop-in shim: ``qfswe`` resolved to the B200 path.

With ``PYTHONPATH=pkg/src`` the reference's import paths (``qfswe.mesh``,
``qfswe.scenario``, ``qfswe.tensors``, ``qfswe.symbolic``, ``qfswe.solver``,
``qfswe.harness``) resolve to ``paper_1904_08684_b200``'s modules, whose
per-stage path runs in the sm_100a kernels.
"""

import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_1904_08684_b200 import harness, mesh, scenario, solver, symbolic, tensors  # noqa: E402

for _name, _mod in (("mesh", mesh), ("scenario", scenario), ("tensors", tensors),
                    ("symbolic", symbolic), ("solver", solver), ("harness", harness)):
    sys.modules[f"{__name__}.{_name}"] = _mod
