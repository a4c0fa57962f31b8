"""Physical scenarios: constants, bathymetry, analytic data, forcing.

Mirrors reference ``qfswe.scenario`` (scenario.py:21-221): a ``Scenario``
dataclass with the same fields (g, f_c, tau_bf, dt, t_end, h_min, hb_mode,
dirichlet_markers, hb, exact, forcing) and ``exact_with_velocity``, plus the
reference builders ``perturbed_square_scenario``, ``ring_scenario``,
``lake_at_rest_scenario`` and ``load_config``/``RunConfig``.

The stage kernels evaluate Dirichlet data and manufactured forcing on the
device every stage, so each scenario also carries
a ``DeviceScenario``: a closed-form family id plus its parameters, with the
derivatives written out by hand (no SymPy at run time).  The host numpy
callables below use the same closed forms and are checked against the
reference's SymPy derivation (scenario.py:69-94) in the tests.

Extensions for the BASELINE configurations:

* ``mms_scenario``: xi = A sin 2pi(x+y-t), u = a cos 2pi(x-t), v = b sin 2pi(y-t),
  U = H u, V = H v over h_b = h0 + hx x + hy y + hxy x y.  It violates the
  sourceless mass equation, which the reference rejects (scenario.py:72-77),
  so a mass source S_xi = xi_t + U_x + V_y is added to the xi equation.
* ``bump_scenario``: seeded Gaussian bumps over seeded sine bathymetry,
  reflective walls, CFL time step.
* ``wall_markers``: boundary markers treated as reflective walls.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable

import numpy as np

__all__ = [
    "Scenario",
    "DeviceScenario",
    "perturbed_square_scenario",
    "ring_scenario",
    "lake_at_rest_scenario",
    "mms_scenario",
    "bump_scenario",
    "custom_scenario",
    "RunConfig",
    "load_config",
    "KIND_NONE",
    "KIND_MMS",
    "KIND_TRAVEL",
    "KIND_LAKE",
    "KIND_USER",
    "user_device_source",
]

TWO_PI = 2.0 * math.pi

# device scenario families (must match csrc/qf_scenario.cuh)
KIND_NONE, KIND_MMS, KIND_TRAVEL, KIND_LAKE, KIND_USER = 0, 1, 2, 3, 4
N_PARAMS = 8


@dataclass(frozen=True)
class DeviceScenario:
    """Closed-form family evaluated inside the stage kernel.

    params (all families): [0..3] = h_b coefficients h0, hx, hy, hxy of
    h_b = h0 + hx x + hy y + hxy x y; the rest is family specific:
      MMS:    [4] A_xi, [5] A_u, [6] A_v
      TRAVEL: [4] C_a, [5] C_t, [6] y_a
      LAKE:   [4] xi0
    """

    kind: int = KIND_NONE
    params: tuple = (0.0,) * N_PARAMS
    has_forcing: bool = False

    def as_array(self) -> np.ndarray:
        p = np.zeros(N_PARAMS)
        p[: len(self.params)] = self.params
        return p


@dataclass
class Scenario:
    """Run physics (reference scenario.py:34-55) plus device descriptor."""

    name: str
    g: float = 9.81
    f_c: float = 0.0
    tau_bf: float = 0.0
    dt: float = 0.5
    t_end: float = 1500.0
    h_min: float = 1e-3
    hb_mode: str = "linear"
    dirichlet_markers: frozenset = frozenset({1})
    hb: Callable = None
    exact: Callable | None = None
    forcing: Callable | None = None
    # --- extensions ---------------------------------------------------
    mass_source: Callable | None = None      # (x, y, t) -> S_xi
    initial: Callable | None = None          # (x, y) -> (xi, U, V), non-analytic data
    wall_markers: frozenset = frozenset()
    cfl: float | None = None                 # dt = cfl * h_min / lambda_max(t=0)
    device: DeviceScenario = field(default_factory=DeviceScenario)

    bump_params: dict | None = None          # drawn bump/mode parameters (bump_scenario)
    # what the device family was built from (a field, so dataclasses.replace keeps it)
    _device_sig: tuple | None = field(default=None, repr=False, compare=False)

    def field_program(self) -> np.ndarray | None:
        """Device field program for qf_project (csrc/qf_kernels.cu), or None."""
        if self.bump_params is not None:
            bp = self.bump_params
            modes = np.column_stack([bp["kv"], bp["ph"]]).ravel()
            bumps = np.column_stack([bp["A"], bp["sig"], bp["cen"]]).ravel()
            head = [1.0, 1.0, len(bp["ph"]), len(bp["A"]), 1.0, 0.2]
            return np.concatenate([head, modes, bumps]).astype(np.float64)
        if self.device.kind not in (KIND_NONE, KIND_USER) and self.initial is None:
            return np.zeros(6)
        return None

    def _physics_signature(self) -> tuple:
        """The callables and constants a device descriptor was built from."""
        return (self.hb, self.exact, self.forcing, self.mass_source, float(self.g),
                float(self.tau_bf), float(self.f_c))

    def _bind_device(self, dev: "DeviceScenario") -> None:
        """Attach a closed-form device family and record what it was built
        from (see ``device_matches``)."""
        self.device = dev
        self._device_sig = self._physics_signature()

    def device_matches(self) -> bool:
        """False when ``hb`` / ``exact`` / ``forcing`` / ``mass_source`` / g /
        tau_bf / f_c were changed after the family factory built the device
        descriptor (the reference itself assigns ``scn.exact`` / ``scn.forcing``
        after construction): the kernels would then evaluate other physics
        than the host callables."""
        sig = self._device_sig
        if sig is None:
            return self.device.kind == KIND_NONE
        cur = self._physics_signature()
        return all(a is b for a, b in zip(sig[:4], cur[:4])) and sig[4:] == cur[4:]

    def exact_with_velocity(self, x, y, t):
        """Analytic (xi, U, V, u, v); u = U/H with H = hb + xi."""
        xi, U, V = self.exact(x, y, t)
        H = self.hb(x, y) + xi
        return xi, U, V, U / H, V / H


# ------------------------------------------------------------- closed forms

def _bilinear_hb(h0, hx, hy, hxy):
    def hb(x, y):
        x = np.asarray(x, dtype=float)
        y = np.asarray(y, dtype=float)
        return h0 + hx * x + hy * y + hxy * x * y
    return hb


def _flux_forcing(g, tau, fc, H, Hx, Hy, U, Ut, Ux, Uy, V, Vt, Vx, Vy, xix, xiy):
    """Momentum forcing of reference scenario.py:78-93 from field derivatives:
    Fx = U_t + (U^2/H)_x + (UV/H)_y + tau U - fc V + g H xi_x, Fy alike."""
    iH = 1.0 / H
    uu, vv = U * iH, V * iH
    Fx = (Ut + 2.0 * uu * Ux - uu * uu * Hx + (Uy * V + U * Vy) * iH - uu * vv * Hy
          + tau * U - fc * V + g * H * xix)
    Fy = (Vt + (Ux * V + U * Vx) * iH - uu * vv * Hx + 2.0 * vv * Vy - vv * vv * Hy
          + tau * V + fc * U + g * H * xiy)
    return Fx, Fy


def _mms_fields(A, au, av, hbp):
    h0, hx, hy, hxy = hbp

    def parts(x, y, t):
        x = np.asarray(x, dtype=float)
        y = np.asarray(y, dtype=float)
        s1, c1 = np.sin(TWO_PI * (x + y - t)), np.cos(TWO_PI * (x + y - t))
        s2, c2 = np.sin(TWO_PI * (x - t)), np.cos(TWO_PI * (x - t))
        s3, c3 = np.sin(TWO_PI * (y - t)), np.cos(TWO_PI * (y - t))
        xi = A * s1
        xit, xix, xiy = -TWO_PI * A * c1, TWO_PI * A * c1, TWO_PI * A * c1
        u, ut, ux = au * c2, TWO_PI * au * s2, -TWO_PI * au * s2
        v, vt, vy = av * s3, -TWO_PI * av * c3, TWO_PI * av * c3
        H = h0 + hx * x + hy * y + hxy * x * y + xi
        Hx, Hy, Ht = hx + hxy * y + xix, hy + hxy * x + xiy, xit
        return dict(xi=xi, xit=xit, xix=xix, xiy=xiy, u=u, ut=ut, ux=ux, v=v, vt=vt,
                    vy=vy, H=H, Hx=Hx, Hy=Hy, Ht=Ht)

    def exact(x, y, t):
        p = parts(x, y, t)
        return p["xi"], p["H"] * p["u"], p["H"] * p["v"]

    def derivs(x, y, t):
        p = parts(x, y, t)
        H, u, v = p["H"], p["u"], p["v"]
        U, V = H * u, H * v
        Ut, Ux, Uy = p["Ht"] * u + H * p["ut"], p["Hx"] * u + H * p["ux"], p["Hy"] * u
        Vt, Vx, Vy = p["Ht"] * v + H * p["vt"], p["Hx"] * v, p["Hy"] * v + H * p["vy"]
        return p, H, U, V, Ut, Ux, Uy, Vt, Vx, Vy

    return exact, derivs


def mms_scenario(amp_xi: float = 0.01, amp_u: float = 0.1, amp_v: float = 0.1,
                 hb_coeffs=(1.0, 0.0, 0.0, 0.1), **kw) -> Scenario:
    """BASELINE C1/C2 manufactured solution on the unit square."""
    exact, derivs = _mms_fields(amp_xi, amp_u, amp_v, hb_coeffs)
    scn = Scenario(name="mms", **kw)
    scn.hb = _bilinear_hb(*hb_coeffs)
    scn.exact = exact
    g, tau, fc = scn.g, scn.tau_bf, scn.f_c

    def forcing(x, y, t):
        p, H, U, V, Ut, Ux, Uy, Vt, Vx, Vy = derivs(x, y, t)
        return _flux_forcing(g, tau, fc, H, p["Hx"], p["Hy"], U, Ut, Ux, Uy,
                             V, Vt, Vx, Vy, p["xix"], p["xiy"])

    def mass_source(x, y, t):
        p, H, U, V, Ut, Ux, Uy, Vt, Vx, Vy = derivs(x, y, t)
        return p["xit"] + Ux + Vy

    scn.forcing = forcing
    scn.mass_source = mass_source
    scn._bind_device(DeviceScenario(KIND_MMS, tuple(hb_coeffs) + (amp_xi, amp_u, amp_v),
                                     has_forcing=True))
    return scn


# reference bench constants (scenario.py:118-131)
BENCH_CA, BENCH_CT, BENCH_YA = 0.2, 0.2, 0.3


def _travel_scenario(name: str, **kw) -> Scenario:
    """Reference travelling wave over h_b = 1 + x/1000 + 2y/1000 (scenario.py:125-141)."""
    Ca, Ct, ya = BENCH_CA, BENCH_CT, BENCH_YA
    hbp = (1.0, 1e-3, 2e-3, 0.0)
    k_ = math.pi / 600.0
    scn = Scenario(name=name, **kw)
    scn.hb = _bilinear_hb(*hbp)

    def parts(x, y, t):
        x = np.asarray(x, dtype=float)
        y = np.asarray(y, dtype=float)
        ph = k_ * (x + y + Ct * t)
        return np.sin(ph), np.cos(ph)

    def exact(x, y, t):
        s, _ = parts(x, y, t)
        return 2 + ya - 2 * Ca * s, 2 * ya + Ca * Ct * s, ya + Ca * Ct * s

    g, tau, fc = scn.g, scn.tau_bf, scn.f_c

    def forcing(x, y, t):
        s, c = parts(x, y, t)
        x = np.asarray(x, dtype=float)
        y = np.asarray(y, dtype=float)
        xi = 2 + ya - 2 * Ca * s
        dxi = -2 * Ca * c * k_                 # d/dx = d/dy; d/dt = Ct * this
        U, V = 2 * ya + Ca * Ct * s, ya + Ca * Ct * s
        dq = Ca * Ct * c * k_
        H = hbp[0] + hbp[1] * x + hbp[2] * y + xi
        return _flux_forcing(g, tau, fc, H, hbp[1] + dxi, hbp[2] + dxi,
                             U, Ct * dq, dq, dq, V, Ct * dq, dq, dq, dxi, dxi)

    scn.exact = exact
    scn.forcing = forcing
    scn._bind_device(DeviceScenario(KIND_TRAVEL, hbp + (Ca, Ct, ya, 0.0), has_forcing=True))
    return scn


def perturbed_square_scenario(**kw) -> Scenario:
    return _travel_scenario("perturbed-square", **kw)


def ring_scenario(**kw) -> Scenario:
    return _travel_scenario("ring", **kw)


def lake_at_rest_scenario(xi0: float = 0.5, slope=(0.001, 0.002),
                          depth: float = 2.0, **kw) -> Scenario:
    """Still water over linear bathymetry (reference scenario.py:144-150)."""
    hbp = (float(depth), float(slope[0]), float(slope[1]), 0.0)
    scn = Scenario(name="lake-at-rest", **kw)
    scn.hb = _bilinear_hb(*hbp)

    def exact(x, y, t):
        shape = np.broadcast(np.asarray(x), np.asarray(y)).shape
        return np.full(shape, float(xi0)), np.zeros(shape), np.zeros(shape)

    scn.exact = exact
    scn.forcing = None
    scn._bind_device(DeviceScenario(KIND_LAKE, hbp + (float(xi0), 0.0, 0.0, 0.0)))
    return scn


def bump_fields(seed: int = 0, n_bumps: int = 16, n_modes: int = 8,
                min_depth: float = 0.25, max_tries: int = 1000):
    """Seeded Gaussian-bump elevation and sine-mode bathymetry (BASELINE C3).

    Draw order from one ``numpy.random.default_rng(seed')`` stream:
    A_j ~ U(0.01, 0.05) (16), sigma_j ~ U(0.02, 0.1) (16), c_j ~ U(0.1, 0.9)^2
    (16 x 2), then |k_j| = 4 pi sqrt(U), angle ~ U(0, 2 pi) (8 each, uniform
    in the disk |k| <= 4 pi), phases ~ U(0, 2 pi) (8).
    xi0 = sum A_j exp(-|x - c_j|^2 / (2 sigma_j^2));
    h_b = 1 + 0.2 sum sin(k_j . x + phi_j).
    Positivity: seed' is the first seed >= ``seed`` whose h_b, sampled on a
    257^2 grid of the unit square, has min >= ``min_depth`` (SURVEY §8d:
    ~29% of raw draws go dry).  Returns (xi0, hb, seed').
    """
    g1 = np.linspace(0.0, 1.0, 257)
    X, Y = np.meshgrid(g1, g1, indexing="ij")
    for s in range(seed, seed + max_tries):
        rng = np.random.default_rng(s)
        A = rng.uniform(0.01, 0.05, n_bumps)
        sig = rng.uniform(0.02, 0.1, n_bumps)
        cen = rng.uniform(0.1, 0.9, (n_bumps, 2))
        kr = 4.0 * math.pi * np.sqrt(rng.uniform(0.0, 1.0, n_modes))
        ka = rng.uniform(0.0, TWO_PI, n_modes)
        kv = np.column_stack([kr * np.cos(ka), kr * np.sin(ka)])
        ph = rng.uniform(0.0, TWO_PI, n_modes)

        def hb(x, y, kv=kv, ph=ph):
            x = np.asarray(x, dtype=float)
            y = np.asarray(y, dtype=float)
            acc = np.zeros(np.broadcast(x, y).shape)
            for j in range(len(ph)):
                acc = acc + np.sin(kv[j, 0] * x + kv[j, 1] * y + ph[j])
            return 1.0 + 0.2 * acc

        if hb(X, Y).min() >= min_depth:
            def xi0(x, y, A=A, sig=sig, cen=cen):
                x = np.asarray(x, dtype=float)
                y = np.asarray(y, dtype=float)
                acc = np.zeros(np.broadcast(x, y).shape)
                for j in range(len(A)):
                    r2 = (x - cen[j, 0]) ** 2 + (y - cen[j, 1]) ** 2
                    acc = acc + A[j] * np.exp(-r2 / (2.0 * sig[j] ** 2))
                return acc
            xi0.params = dict(A=A, sig=sig, cen=cen, kv=kv, ph=ph)
            return xi0, hb, s
    raise ValueError("no admissible bathymetry seed found")


def bump_scenario(seed: int = 0, cfl: float = 0.1, **kw) -> Scenario:
    """BASELINE C3-C5: bumps at rest, reflective walls, dt from CFL."""
    xi0, hb, used = bump_fields(seed)
    kw.setdefault("dirichlet_markers", frozenset())
    kw.setdefault("wall_markers", frozenset({1}))
    scn = Scenario(name=f"bumps-seed{used}", cfl=cfl, **kw)
    scn.hb = hb

    def initial(x, y):
        v = xi0(x, y)
        return v, np.zeros_like(v), np.zeros_like(v)

    scn.initial = initial
    scn.bump_params = xi0.params
    scn.device = DeviceScenario(KIND_NONE)
    return scn


def custom_scenario(xi: str, U: str, V: str, hb: str, **kw) -> Scenario:
    """Scenario from SymPy expression strings in x, y, t (reference
    scenario.py:153-157, built like ``_build(..., manufacture=True)``): host
    callables by ``lambdify``, the momentum forcing manufactured from the
    fields (reference ``_manufacture``, scenario.py:69-94; ValueError for a
    non-zero mass residual), and a device description that
    ``Discretization`` compiles into a per-scenario module
    (``device_source``, csrc/qf_user.cuh, ``qf_user_scenario``): Dirichlet
    data and forcing are evaluated on the GPU every stage, like the reference
    evaluates ``exact_with_velocity`` and ``forcing`` (solver.py:396,637,721).
    """
    import sympy as sp

    X, Y, T = sp.symbols("x y t", real=True)
    loc = {"x": X, "y": Y, "t": T}
    ex = [sp.sympify(s, locals=loc) for s in (xi, U, V, hb)]
    scn = Scenario(name="custom", **kw)
    xi_e, U_e, V_e, hb_e = ex
    H = hb_e + xi_e
    residual = sp.simplify(sp.diff(xi_e, T) + sp.diff(U_e, X) + sp.diff(V_e, Y))
    if residual != 0:
        raise ValueError(f"analytic fields violate the sourceless mass equation: residual {residual}")
    g = sp.Float(scn.g)
    Fx = (sp.diff(U_e, T) + sp.diff(U_e**2 / H, X) + sp.diff(U_e * V_e / H, Y)
          + scn.tau_bf * U_e - scn.f_c * V_e + g * H * sp.diff(xi_e, X))
    Fy = (sp.diff(V_e, T) + sp.diff(U_e * V_e / H, X) + sp.diff(V_e**2 / H, Y)
          + scn.tau_bf * V_e + scn.f_c * U_e + g * H * sp.diff(xi_e, Y))

    def lam(args, exprs):
        fns = [sp.lambdify(args, e, modules="numpy") for e in exprs]

        def call(*vals):
            shape = np.broadcast(*[np.asarray(v) for v in vals]).shape
            return tuple(np.broadcast_to(np.asarray(f(*vals), dtype=float), shape) for f in fns)
        return call

    f_hb = lam((X, Y), [hb_e])
    scn.hb = lambda x, y: f_hb(x, y)[0]
    scn.exact = lam((X, Y, T), ex[:3])
    manufactured = not (Fx == 0 and Fy == 0)
    scn.forcing = lam((X, Y, T), [Fx, Fy]) if manufactured else None
    scn._custom_exprs = ex  # type: ignore[attr-defined]
    scn._custom_syms = (X, Y, T)  # type: ignore[attr-defined]
    scn._custom_forcing = (Fx, Fy) if manufactured else None  # type: ignore[attr-defined]
    scn._bind_device(DeviceScenario(KIND_USER, has_forcing=manufactured))
    return scn


def user_device_source(scn: Scenario, k: int) -> str:
    """CUDA source of a custom scenario's device module for order k: the
    SymPy fields printed as C99 (common subexpressions shared), wrapped in
    the templates of csrc/qf_user.cuh."""
    import sympy as sp
    from sympy.printing.c import C99CodePrinter

    pr = C99CodePrinter()

    def body(outs, exprs):
        reps, red = sp.cse([sp.sympify(e) for e in exprs], symbols=sp.numbered_symbols("q_"))
        lines = [f"    const double {s} = {pr.doprint(e)};" for s, e in reps]
        lines += [f"    {o} = {pr.doprint(e)};" for o, e in zip(outs, red)]
        return "\n".join(lines)

    xi, U, V, hb = scn._custom_exprs
    F = scn._custom_forcing or (sp.Integer(0), sp.Integer(0))
    return f"""// generated by paper_1904_08684_b200/scenario.py:user_device_source (k = {k})
#include <math.h>
#ifndef M_PI
#define M_PI 3.141592653589793
#endif
#include "qf_device.cuh"
#include "generated/qf_order{k}.cuh"
#include "qf_user.cuh"
struct UserScn {{
  static __device__ void exact(double x, double y, double t, double& xi, double& U, double& V,
                               double& hb) {{
{body(("xi", "U", "V", "hb"), (xi, U, V, hb))}
  }}
  static __device__ void forcing(double x, double y, double t, double& Fx, double& Fy) {{
{body(("Fx", "Fy"), F)}
  }}
}};
extern "C" __global__ void __launch_bounds__(128) qf_user_ghost(
    qf::Tab T, const int* bel, const int* bloc, int nb, int nstage, double t0,
    const double* t_dev, double3 toffs, double* ghost) {{
  qf::user_ghost<{k}, UserScn>(T, bel, bloc, nb, nstage, t0, t_dev, toffs, ghost);
}}
extern "C" __global__ void __launch_bounds__(128) qf_user_forcing(
    qf::Tab T, const double* t_dev, double t0, double toff, int e0, int n, double* frc) {{
  qf::user_forcing<{k}, UserScn>(T, t_dev, t0, toff, e0, n, frc);
}}
"""


_SCENARIOS = {
    "perturbed-square": perturbed_square_scenario,
    "ring": ring_scenario,
    "lake-at-rest": lake_at_rest_scenario,
    "mms": mms_scenario,
    "bumps": bump_scenario,
}


@dataclass
class RunConfig:
    """Parsed run configuration (reference scenario.py:167-191)."""

    scenario: Scenario
    order: int
    mesh_spec: dict
    output: dict = field(default_factory=dict)

    def build_mesh(self):
        from .mesh import build_ring_mesh, build_square_mesh, build_unit_square_mesh, load_mesh

        ms = self.mesh_spec
        if "path" in ms:
            return load_mesh(ms["path"])
        gen = ms.get("generator", "square")
        if gen == "square":
            return build_square_mesh(level=int(ms.get("level", 2)),
                                     perturb=float(ms.get("perturb", 0.0)),
                                     seed=int(ms.get("seed", 0)))
        if gen == "ring":
            return build_ring_mesh(level=int(ms.get("level", 2)))
        if gen == "unit-square":
            return build_unit_square_mesh(int(ms.get("n", 32)), float(ms.get("jitter", 0.0)),
                                          int(ms.get("seed", 0)))
        raise ValueError(f"unknown mesh generator {gen!r}")


def load_config(path) -> RunConfig:
    """JSON config (reference scenario.py:194-221) plus 'mms'/'bumps'/'unit-square'."""
    with open(path) as fh:
        cfg = json.load(fh)
    name = cfg.get("scenario", "perturbed-square")
    physics = cfg.get("physics", {})
    kw = dict(g=float(physics.get("g", 9.81)), f_c=float(physics.get("f_c", 0.0)),
              tau_bf=float(physics.get("tau_bf", 0.0)),
              h_min=float(physics.get("h_min", 1e-3)), dt=float(cfg.get("dt", 0.5)),
              t_end=float(cfg.get("t_end", 1500.0)), hb_mode=cfg.get("hb_mode", "linear"))
    if name == "custom":
        f = cfg["fields"]
        scn = custom_scenario(f["xi"], f["U"], f["V"], f["hb"], **kw)
    elif name in _SCENARIOS:
        scn = _SCENARIOS[name](**kw)
    else:
        raise ValueError(f"unknown scenario {name!r}")
    return RunConfig(scenario=scn, order=int(cfg.get("order", 1)),
                     mesh_spec=cfg.get("mesh", {"generator": "square", "level": 2}),
                     output=cfg.get("output", {}))
