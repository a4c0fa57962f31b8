"""B200-native (sm_100a, FP64) per-stage RHS path of the quadrature-free DG
shallow-water solver of arXiv 1904.08684, behind the reference ``qfswe``
mesh / solver / step API.

Host modules mirror the reference package (``mesh``, ``scenario``,
``tensors``, ``symbolic``, ``solver``, ``harness``); the per-stage work runs
in the hand-written kernels of ``csrc/`` through the C ABI of
``include/qfswe.h``.
"""

__version__ = "0.1.0"
