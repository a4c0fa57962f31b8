"""Discretization / State: the reference's solver API on the B200 path.

Drop-in for reference ``qfswe.solver`` (solver.py:28-34, 48-780):
``State(c, u, t)``, ``Discretization(mesh, scenario, order, backend)`` with
``project_volume``, ``project_initial``, ``solve_velocity``,
``compute_lambda``, ``element_rhs``, ``edge_rhs``, ``source_rhs``, ``rhs``,
``step``, ``run`` and the same exceptions (``DryState``,
``SingularProjection``, ``FloatingPointError``, ``ValueError``, CFL
``UserWarning``).

All per-stage work runs in the sm_100a kernels behind the C ABI
(``_cabi.py`` -> ``libqfswe.so``); the state stays device-resident in a
structure-of-arrays layout between steps and ``State.c`` / ``State.u`` are
materialised lazily.  Setup (geometry, quadrature, bathymetry projection)
stays on the host, vectorised in NumPy.  There is no CPU fallback: without
the library or a CUDA device the constructor raises.
"""

from __future__ import annotations

import math
import warnings

import numpy as np

from . import _cabi
from .layout import BND_DIRICHLET, build_tables, pad_ld
from .mesh import ElementGeometry, Mesh, compute_geometry, locality_order
from .scenario import KIND_MMS, KIND_NONE, KIND_USER, Scenario
from .symbolic import build_basis
from .tensors import build_ref_tensors, triangle_rule

__all__ = ["DryState", "SingularProjection", "State", "Discretization", "flux_dot_n",
           "cfl_time_step"]

XI, U, V = 0, 1, 2


class DryState(ArithmeticError):
    """Total water depth at or below the configured minimum."""


class SingularProjection(ArithmeticError):
    """Per-element velocity projection system is numerically singular."""


def cfl_time_step(cfl: float, k: int, h_min: float, lam_max: float) -> float:
    """CFL time step of the BASELINE C3-C5 runs (the reference has none).

    dt = cfl * h_min / ((2k + 1) * lambda_max), with h_min the reference's
    min(detB / longest edge) (solver.py:240-246) and lambda_max the largest
    Lax-Friedrichs speed at t = 0.  The 1/(2k+1) factor is the usual DG
    stability scaling (without it, k = 4 / SSP-RK3 at cfl = 0.1 blows up in
    ~10 steps in both the oracle and the GPU path).
    """
    return float(cfl) * h_min / ((2 * k + 1) * lam_max)


def flux_dot_n(xi, Uq, Vq, uu, uv, hb, n1, n2, g):
    """Pointwise modified flux . n (reference solver.py:60-71), test oracle."""
    pressure = 0.5 * g * xi * (xi + 2.0 * hb)
    return (Uq * n1 + Vq * n2, (Uq * uu + pressure) * n1 + (Uq * uv) * n2,
            (Vq * uu) * n1 + (Vq * uv + pressure) * n2)


class State:
    """Modal coefficients c[e, j, i] (xi, U, V) and u[e, j, i] (u, v) at time t.

    Host arrays are materialised lazily from the device copy; once they are
    handed out the device copy is dropped (the caller may mutate them), so a
    later ``step`` re-uploads.
    """

    def __init__(self, c=None, u=None, t: float = 0.0, _dev=None):
        self._c = c
        self._u = u
        self.t = float(t)
        self._dev = _dev  # (disc, DeviceState)

    def _materialise(self):
        if self._dev is not None and (self._c is None or self._u is None):
            disc, ds = self._dev
            self._c, self._u = disc._download(ds)
            self._dev = None

    @property
    def c(self) -> np.ndarray:
        self._materialise()
        return self._c

    @c.setter
    def c(self, v):
        self._materialise()
        self._c = v

    @property
    def u(self) -> np.ndarray:
        self._materialise()
        return self._u

    @u.setter
    def u(self, v):
        self._materialise()
        self._u = v

    def copy(self) -> "State":
        if self._dev is not None and self._c is None:
            disc, ds = self._dev
            return State(t=self.t, _dev=(disc, ds.clone()))
        return State(self.c.copy(), self.u.copy(), self.t)


class DeviceState:
    """(c, u) in SoA layout on the device plus the device time {t, dt}."""

    def __init__(self, c, u, t_dev):
        self.c, self.u, self.t_dev = c, u, t_dev

    def clone(self) -> "DeviceState":
        return DeviceState(self.c.clone(), self.u.clone(), self.t_dev.clone())


def _on_device(fn):
    """Run a Discretization method with its CUDA device current (torch
    allocations, library launches without a context and the context's own
    entry points all agree on the device)."""
    import functools

    @functools.wraps(fn)
    def wrap(self, *a, **kw):
        with self.torch.cuda.device(self.device):
            return fn(self, *a, **kw)
    return wrap


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the B200 path needs a CUDA device (no CPU fallback)")
    return torch


def _project(vals_w: np.ndarray, phi: np.ndarray) -> np.ndarray:
    """(E, Q) x (P, Q)^T with a fixed per-row summation order (elementwise
    accumulation over q), so an element's coefficients do not depend on how
    many elements are projected together: BLAS GEMM blocking does (k = 4
    P1 bathymetry differed by 1 ulp between a partition and the whole mesh,
    which broke bitwise partition independence)."""
    out = vals_w[:, :1] * phi[:, 0]
    for q in range(1, vals_w.shape[1]):
        out = out + vals_w[:, q:q + 1] * phi[:, q]
    return out


class HostSetup:
    """Host-side (NumPy) setup shared by the device path and the CPU tests:
    geometry, quadrature, P1 bathymetry, SoA tables (reference solver.py:103-270)."""

    #: local element count from which setup projections run on the device
    DEVICE_SETUP_MIN = 1_000_000

    def __init__(self, mesh: Mesh, scenario: Scenario, order: int, backend: str = "einsum",
                 elements=None, n_own: int | None = None, device_setup: bool | None = None,
                 slot_order: str = "locality", halo_code=None, device_tables: bool | None = None):
        """``elements``/``n_own`` restrict the discretization to a partition
        (``distributed.py``): the owned elements, interior first; neighbours
        owned by other partitions are rows of a halo trace table
        (``halo_code[j][slot]``, see ``distributed.Halo``).
        ``device_setup`` moves the initial / bathymetry projections to the GPU
        (``qf_project``; default: automatic for large meshes).  ``slot_order``:
        device element slots in Z-order ("locality", default) or mesh order
        ("natural") or a seeded shuffle ("random", for tests: every neighbour out
        of block); results are identical, only the memory locality differs.
        ``device_tables`` builds connectivity, geometry, Z-order slots and the
        SoA tables on the GPU (``device_setup.py``; default: with
        ``device_setup`` on a whole mesh); host geometry and connectivity are
        then computed only if an API asks for them."""
        if slot_order not in ("locality", "natural", "random"):
            raise ValueError("slot_order must be 'locality', 'natural' or 'random'")
        self.slot_order = slot_order
        if backend not in ("einsum", "ir"):
            raise ValueError("backend must be 'einsum' or 'ir'")
        if scenario.hb_mode not in ("linear", "const"):
            raise ValueError("hb_mode must be 'linear' or 'const'")
        self.mesh = mesh
        self.scn = scenario
        self.k = int(order)
        self.backend = backend  # accepted for signature compatibility only
        self.basis = build_basis(self.k)
        self.K = self.basis.size
        self._geom = self._edge_geom = None
        self.partitioned = elements is not None
        if elements is None:
            self.elements = np.arange(mesh.n_triangles)
            self.n_own = mesh.n_triangles
        else:
            self.elements = np.asarray(elements, dtype=np.int64)
            self.n_own = len(self.elements) if n_own is None else int(n_own)
        prog = scenario.field_program()
        if device_setup is None:
            device_setup = prog is not None and len(self.elements) >= self.DEVICE_SETUP_MIN
        if device_setup and prog is None:
            raise ValueError(f"scenario {scenario.name!r} has no device field program")
        self.device_setup = bool(device_setup)
        if device_tables is None:
            device_tables = self.device_setup and not self.partitioned and slot_order == "locality"
        self.device_tables = bool(device_tables)
        self._nh = 1 if self.k == 0 else 3
        self._setup_quadrature()
        if not self.device_setup:
            self._setup_bathymetry()
        self._perm_host = None
        if self.device_tables:
            from .device_setup import device_tables as build_device_tables
            import torch

            if self.partitioned or slot_order != "locality":
                raise ValueError("device tables are built for whole meshes in Z-order slots")
            self.tables = build_device_tables(mesh, scenario.dirichlet_markers,
                                              scenario.wall_markers,
                                              torch.device("cuda", torch.cuda.current_device()))
            self.setup_seconds = self.tables.seconds
        else:
            # device slot order: locality (Z-order) permutation of the local rows
            # for a whole mesh; a partition's local order is already sorted
            if self.partitioned or self.slot_order == "natural":
                self._perm_host = None
            elif self.slot_order == "random":
                self._perm_host = np.random.default_rng(0).permutation(mesh.n_triangles)
            else:
                self._perm_host = locality_order(mesh)
            slots = self.elements if self._perm_host is None else self.elements[self._perm_host]
            self.tables = build_tables(mesh, scenario.dirichlet_markers, scenario.wall_markers,
                                       slots, self.n_own, halo_code=halo_code)
        self.h_min = self.tables.h_min
        if not scenario.device_matches():
            raise ValueError(f"scenario {scenario.name!r}: hb / exact / forcing / mass_source / g / "
                             "tau_bf / f_c were changed after its device family was built; the "
                             "kernels would evaluate different physics than the host callables "
                             "(build a new scenario instead)")
        needs_data = int(self.tables.bnd_elem.shape[0]) > 0 or scenario.forcing is not None \
            or scenario.mass_source is not None
        if needs_data and scenario.device.kind == KIND_NONE:
            raise ValueError(f"scenario {scenario.name!r} needs boundary data or forcing that "
                             "has no device evaluator (use a closed-form scenario family)")
        self._cfl_warned = False
        self.cfl_warn_threshold = 2.0
        # reference solver.py:123-124: per-interior-edge xi mass flux of the
        # left / right element, recorded by edge_rhs / rhs when enabled
        self.instrument_mass_flux: bool = False
        self.last_mass_flux: tuple | None = None
        self.dt = scenario.dt
        self._dt_fixed = scenario.cfl is None
        self.phi_at_vertices = np.array(
            [[f.eval_point(*v) for v in ((0.0, 0.0), (1.0, 0.0), (0.0, 1.0))]
             for f in self.basis.functions])

    # ------------------------------------------------------------- setup
    @property
    def perm(self):
        """Device slot -> local element row (None: identity); host copy."""
        if self.device_tables and self._perm_host is None:
            self._perm_host = self.tables.perm.cpu().numpy()
        return self._perm_host

    def _host_geometry(self):
        geom, self._edge_geom = compute_geometry(self.mesh)
        if self.partitioned:
            el = self.elements
            geom = ElementGeometry(B=geom.B[el], detB=geom.detB[el],
                                   sqrt_detB=geom.sqrt_detB[el], a1=geom.a1[el])
        self._geom = geom

    @property
    def geom(self) -> ElementGeometry:
        """Host element geometry (reference mesh.py:259-282), built on first use."""
        if self._geom is None:
            self._host_geometry()
        return self._geom

    @property
    def edge_geom(self):
        if self._edge_geom is None:
            self._host_geometry()
        return self._edge_geom

    @property
    def tensors(self):
        """Reference-form tensors (exact; lazily built, not used by the kernels)."""
        return build_ref_tensors(self.k)

    def _setup_quadrature(self):
        pts, wts = triangle_rule(2 * self.k + 2)
        self.quad_ref, self.quad_w = pts, wts
        self.quad_phi = np.array([f.eval(pts[:, 0], pts[:, 1]) for f in self.basis.functions])
        self._quad_xy = None

    @property
    def quad_xy(self) -> np.ndarray:
        """(E, Q, 2) physical quadrature points (built on first use)."""
        if self._quad_xy is None:
            B, a1 = self.geom.B, self.geom.a1
            self._quad_xy = np.einsum("eab,qb->eqa", B, self.quad_ref) + a1[:, None, :]
        return self._quad_xy

    def _setup_bathymetry(self):
        """P1 projection of h_b and its constant gradient (solver.py:139-168)."""
        sd = self.geom.sqrt_detB
        vals = self.scn.hb(self.quad_xy[:, :, 0], self.quad_xy[:, :, 1])
        keep = 1 if self.k == 0 else 3
        proj = sd[:, None] * _project(vals * self.quad_w, self.quad_phi[:keep])
        self.hb_coef = np.zeros((len(sd), self.K))
        self.hb_coef[:, :keep] = proj
        if keep == 3:
            g1 = np.array([float(self.basis.gradients[i][0].eval(0.0, 0.0)) for i in range(3)])
            g2 = np.array([float(self.basis.gradients[i][1].eval(0.0, 0.0)) for i in range(3)])
            d1, d2 = proj @ g1, proj @ g2
            B, det = self.geom.B, self.geom.detB
            sc = det * sd
            self.hb_grad = np.column_stack([(B[:, 1, 1] * d1 - B[:, 1, 0] * d2) / sc,
                                            (-B[:, 0, 1] * d1 + B[:, 0, 0] * d2) / sc])
        else:
            self.hb_grad = np.zeros((len(sd), 2))
        self.hb_mean = self.hb_coef[:, 0] / (math.sqrt(2.0) * sd)

    def project_fields(self) -> np.ndarray:
        """Initial (xi, U, V) coefficients of every local element (owned + halo)."""
        scn = self.scn
        x, y = self.quad_xy[:, :, 0], self.quad_xy[:, :, 1]
        if scn.initial is not None:
            fields = scn.initial(x, y)
        elif scn.exact is not None:
            fields = scn.exact(x, y, 0.0)
        else:
            raise ValueError("scenario has no analytic solution to project")
        sd = self.geom.sqrt_detB[:, None]
        c = np.stack([sd * _project(f * self.quad_w, self.quad_phi) for f in fields], axis=1)
        H = (self.hb_coef + c[:, XI]) @ self.quad_phi / self.geom.sqrt_detB[:, None]
        if (H < scn.h_min).any():
            raise DryState(f"projected depth fell below h_min = {scn.h_min}")
        return c

    def hb_table(self) -> np.ndarray:
        """[NH][ld] bathymetry rows of the SoA layout (host setup path)."""
        hb = np.zeros((self._nh, self.tables.ld))
        rows = self.hb_coef if self.perm is None else self.hb_coef[self.perm]
        hb[:, : len(self.elements)] = rows[:, : self._nh].T
        return hb


class Discretization(HostSetup):
    """Mesh + order + scenario bound to device tables (reference solver.py:100-124)."""

    def __init__(self, mesh: Mesh, scenario: Scenario, order: int, backend: str = "einsum",
                 device: int | None = None, elements=None, n_own: int | None = None,
                 device_setup: bool | None = None, slot_order: str = "locality", halo_code=None,
                 device_tables: bool | None = None):
        if device is not None:  # device tables and projections on that device
            import torch
            with torch.cuda.device(device):
                super().__init__(mesh, scenario, order, backend, elements, n_own, device_setup,
                                 slot_order, halo_code, device_tables)
        else:
            super().__init__(mesh, scenario, order, backend, elements, n_own, device_setup,
                             slot_order, halo_code, device_tables)
        self._setup_device(device)

    def _setup_device(self, device):
        torch = _torch()
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self._pin_in = None      # persistent pinned staging of host State.c uploads
        self._pin_in_ev = None   # its last H2D (the buffer is reused after it completes)
        with torch.cuda.device(self.device):
            self._setup_device_tables()

    def _setup_device_tables(self):
        torch = self.torch
        lib = _cabi.load()
        tb = self.tables
        E, ld = tb.n_elem, tb.ld
        self.ld = ld
        dev = self.device
        on = (lambda a: a.to(dev)) if self.device_tables else \
            (lambda a: torch.from_numpy(a).to(dev))  # noqa: E731
        self._geo = on(tb.geo)
        if self.device_setup:
            self._hb = torch.zeros((self._nh, ld), dtype=torch.float64, device=dev)
        else:
            self._hb = torch.from_numpy(self.hb_table()).to(dev)
        self._nbr = on(tb.nbr)
        nb = int(tb.bnd_elem.shape[0])
        if self.device_tables:
            self._perm = tb.perm.to(torch.int32)
        else:
            self._perm = None if self.perm is None else \
                torch.from_numpy(self.perm.astype(np.int32)).to(dev)
        self._bel = on(tb.bnd_elem)
        self._bloc = on(tb.bnd_local)
        self._ghost = torch.zeros(3 * max(nb, 1) * (5 * (self.k + 2) + 6), dtype=torch.float64,
                                  device=dev)
        scn = self.scn
        d = _cabi.QfDesc()
        d.order, d.n_elem, d.ld = self.k, E, ld
        d.geo, d.hb, d.nbr = self._geo.data_ptr(), self._hb.data_ptr(), self._nbr.data_ptr()
        d.n_bnd = nb
        d.bnd_elem, d.bnd_local = self._bel.data_ptr(), self._bloc.data_ptr()
        d.ghost = self._ghost.data_ptr()
        self._hbt = torch.zeros((3 * (self.k + 1) + 1, ld), dtype=torch.float64, device=dev)
        d.hbt = self._hbt.data_ptr()
        d.g, d.f_c, d.tau_bf = scn.g, scn.f_c, scn.tau_bf
        d.hb_linear = 1 if scn.hb_mode == "linear" else 0
        d.scn_kind = scn.device.kind
        for i, p in enumerate(scn.device.as_array()):
            d.scn_params[i] = float(p)
        user = scn.device.kind == KIND_USER
        # (user scenarios: forcing and boundary data come from their own module)
        d.has_forcing = 0 if user else \
            (1 if (scn.forcing is not None or scn.mass_source is not None) else 0)
        # element-local Taylor sin/cos for the MMS phases: 1 = degree 9/8
        # (|z| <= 0.06), 2 = degree 7/6 (|z| <= 0.02); truncation < 1e-18
        ang = self._max_quad_angle() if scn.device.kind == KIND_MMS else 1.0
        d.taylor = 2 if ang <= 0.02 else (1 if ang <= 0.06 else 0)
        uni = self._uniform_phase_table() if d.has_forcing else None
        self._uni = None if uni is None else torch.from_numpy(uni).to(dev)
        d.uni = None if uni is None else self._uni.data_ptr()
        self._desc = d
        ctx = _cabi.C.c_void_p()
        _cabi.check(lib.qf_create(_cabi.C.byref(d), _cabi.C.byref(ctx)), "qf_create")
        self._ctx = ctx
        self._lib = lib
        self._work = None
        if user:
            self._load_user_module()
        if not self.device_setup:
            self._check(lib.qf_static(ctx, len(self.elements), self._stream), "qf_static")
        if self.device_setup:
            self._prog = torch.from_numpy(self.scn.field_program()).to(dev)
            c0, _ = self._empty_state()
            c0.zero_()
            self._check(lib.qf_project(ctx, self._prog.data_ptr(), len(self.elements),
                                       float(self.scn.h_min), c0.data_ptr(), self._hb.data_ptr(),
                                       self._stream), "qf_project")
            self._c_init = c0
            self._raise_errors("initial projection")

    def _load_user_module(self):
        """Compile and bind the custom scenario's device module (Dirichlet
        data + manufactured forcing, csrc/qf_user.cuh)."""
        from .build import compile_user_module
        from .scenario import user_device_source

        image = compile_user_module(user_device_source(self.scn, self.k))
        self._user_image = _cabi.C.create_string_buffer(image, len(image))
        forcing = self.scn.forcing is not None
        _cabi.check(self._lib.qf_user_scenario(self._ctx, self._user_image, len(image),
                                               1 if forcing else 0), "qf_user_scenario")

    def _uniform_phase_table(self):
        """MMS forcing on a mesh whose element Jacobians take at most two
        values (the BASELINE split-square meshes at N = 2^j): sin/cos of the
        per-point phase offsets 2 pi B (r_q - centroid) per Jacobian class,
        so the kernel only rotates the centroid phases (qfswe.h ``uni``).
        None when the mesh has more than two Jacobians or k > 2."""
        if self.k > 2 or self.scn.device.kind != KIND_MMS:
            return None
        n = self.tables.n_elem
        geo = self.tables.host("geo")[:4, :n] if self.device_tables else self.tables.geo[:4, :n]
        if n == 0:
            return None
        cls = np.unique(geo.T, axis=0)
        if len(cls) > 2:
            return None
        B1 = cls[-1]
        nq = len(self.quad_ref)
        r = self.quad_ref - 1.0 / 3.0
        tab = np.zeros(8 + 2 * (6 * nq + 2))
        tab[:4] = B1
        for c, Bc in enumerate((cls[0], B1)):
            z = 2.0 * math.pi * (Bc[0] * r[:, 0] + Bc[1] * r[:, 1])
            w = 2.0 * math.pi * (Bc[2] * r[:, 0] + Bc[3] * r[:, 1])
            rows = np.stack([np.sin(z), np.cos(z), np.sin(w), np.cos(w),
                             np.sin(z + w), np.cos(z + w)], axis=1)
            o = 8 + c * (6 * nq + 2)
            tab[o:o + 6 * nq] = rows.ravel()
        return tab

    def _max_quad_angle(self) -> float:
        """max |2 pi (x_q - x_centroid)| over quadrature points (MMS Taylor gate)."""
        B = self.geom.B
        r = self.quad_ref - 1.0 / 3.0
        d = np.abs(np.einsum("eab,qb->eqa", B, r)).max() if len(B) else 0.0
        return 2.0 * math.pi * float(d)

    def __del__(self):
        try:
            if getattr(self, "_ctx", None):
                self._lib.qf_destroy(self._ctx)
                self._ctx = None
        except Exception:
            pass

    # ------------------------------------------------------- device state
    @property
    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def _perm_ptr(self, n: int):
        """Device slot -> host row map for pack/unpack (None: identity)."""
        if self._perm is None:
            return None
        if n != len(self._perm):
            raise ValueError("permuted layout needs full-length host arrays")
        return self._perm.data_ptr()

    @_on_device
    def upload_fields(self, arr: np.ndarray):
        """(n, F, K) host array (n <= local elements) -> device SoA [F][K][ld]."""
        t = self.torch
        n, F, _ = arr.shape
        a = t.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(self.device)
        out = t.zeros((F, self.K, self.ld), dtype=t.float64, device=self.device)
        _cabi.check(self._lib.qf_pack(a.data_ptr(), out.data_ptr(), n, F, self.K, self.ld,
                                      self._perm_ptr(n), self._stream), "qf_pack")
        return out

    def _empty_state(self):
        t = self.torch
        return (t.empty((3, self.K, self.ld), dtype=t.float64, device=self.device),
                t.empty((2, self.K, self.ld), dtype=t.float64, device=self.device))

    def _pinned_host(self, c_host: np.ndarray):
        """A pinned host tensor holding ``c_host``: the array itself when it
        already lives in page-locked memory (States returned by this class
        are), else a copy in the persistent staging buffer (no per-call
        page-locking)."""
        t = self.torch
        h = t.from_numpy(np.ascontiguousarray(c_host, dtype=np.float64))
        if h.is_pinned():
            return h
        if self._pin_in is None or self._pin_in.shape != h.shape:
            self._pin_in = t.empty(h.shape, dtype=t.float64, pin_memory=True)
            self._pin_in_ev = None
        if self._pin_in_ev is not None:
            self._pin_in_ev.synchronize()  # previous upload from the buffer has finished
        self._pin_in.copy_(h)
        return self._pin_in

    @_on_device
    def _upload_c(self, c_host: np.ndarray):
        t = self.torch
        E = len(c_host)
        h = self._pinned_host(c_host)
        a = h.to(self.device, non_blocking=True)
        if h is self._pin_in:
            self._pin_in_ev = t.cuda.Event()
            self._pin_in_ev.record(t.cuda.current_stream(self.device))
        c, _ = self._empty_state()
        c.zero_()
        _cabi.check(self._lib.qf_pack(a.data_ptr(), c.data_ptr(), E, a.shape[1], self.K, self.ld,
                                      self._perm_ptr(E), self._stream), "qf_pack")
        return c

    @_on_device
    def _download(self, ds: DeviceState):
        t = self.torch
        E = self.tables.n_elem
        ca = t.empty((E, 3, self.K), dtype=t.float64, device=self.device)
        ua = t.empty((E, 2, self.K), dtype=t.float64, device=self.device)
        s = self._stream
        pp = self._perm_ptr(E)
        _cabi.check(self._lib.qf_unpack(ds.c.data_ptr(), ca.data_ptr(), E, 3, self.K, self.ld, pp,
                                        s), "qf_unpack")
        _cabi.check(self._lib.qf_unpack(ds.u.data_ptr(), ua.data_ptr(), E, 2, self.K, self.ld, pp,
                                        s), "qf_unpack")
        # page-locked destinations (torch's caching host allocator recycles
        # them once the arrays are dropped): one async D2H each, one sync; the
        # returned arrays are caller-owned and feed the next upload directly
        hc = t.empty(ca.shape, dtype=t.float64, pin_memory=True)
        hu = t.empty(ua.shape, dtype=t.float64, pin_memory=True)
        hc.copy_(ca, non_blocking=True)
        hu.copy_(ua, non_blocking=True)
        t.cuda.current_stream(self.device).synchronize()
        return hc.numpy(), hu.numpy()

    @_on_device
    def _soa_to_host(self, x, F):
        t = self.torch
        E = self.tables.n_elem
        a = t.empty((E, F, self.K), dtype=t.float64, device=self.device)
        _cabi.check(self._lib.qf_unpack(x.data_ptr(), a.data_ptr(), E, F, self.K, self.ld,
                                        self._perm_ptr(E), self._stream), "qf_unpack")
        return a.cpu().numpy()

    @_on_device
    def to_device(self, state: State, solve: bool = True) -> DeviceState:
        """Device copy of ``state`` (re-used when the state came from the device)."""
        if state._dev is not None and state._c is None and state._dev[0] is self:
            return state._dev[1]
        c = self._upload_c(state.c)
        _, u = self._empty_state()
        u.zero_()
        if solve:
            self._check(self._lib.qf_velocity(self._ctx, c.data_ptr(), u.data_ptr(), 0, -1,
                                              self._stream), "qf_velocity")
        tdev = self.torch.tensor([state.t, self.dt], dtype=self.torch.float64, device=self.device)
        return DeviceState(c, u, tdev)

    def _check(self, status, what):
        _cabi.check(status, what)

    @_on_device
    def _raise_errors(self, where: str):
        bits = _cabi.C.c_uint32(0)
        _cabi.check(self._lib.qf_error(self._ctx, _cabi.C.byref(bits), 1, self._stream),
                    "qf_error")
        b = bits.value
        if b & _cabi.BIT_DRY:
            raise DryState(f"non-positive depth at an edge sample ({where})")
        if b & _cabi.BIT_SINGULAR:
            raise SingularProjection(f"velocity projection is singular ({where})")
        if b & _cabi.BIT_NONFINITE:
            raise FloatingPointError(f"non-finite state ({where})")

    # ------------------------------------------------- projection helpers
    def project_volume(self, fn, t: float | None = None) -> np.ndarray:
        x, y = self.quad_xy[:, :, 0], self.quad_xy[:, :, 1]
        vals = fn(x, y) if t is None else fn(x, y, t)
        return self.geom.sqrt_detB[:, None] * ((vals * self.quad_w) @ self.quad_phi.T)

    @_on_device
    def _device_initial(self) -> DeviceState:
        c = self._c_init.clone()
        _, u = self._empty_state()
        u.zero_()
        self._check(self._lib.qf_velocity(self._ctx, c.data_ptr(), u.data_ptr(), 0,
                                          len(self.elements), self._stream), "qf_velocity")
        tdev = self.torch.tensor([0.0, self.dt], dtype=self.torch.float64, device=self.device)
        return DeviceState(c, u, tdev)

    @_on_device
    def lambda_max(self, ds: DeviceState, t: float = 0.0) -> float:
        """max over owned element edges of the LF speed of a device state."""
        lam = self.torch.zeros((3, self.ld), dtype=self.torch.float64, device=self.device)
        out, _ = self._empty_state()
        self._check(self._lib.qf_rhs(self._ctx, ds.c.data_ptr(), ds.u.data_ptr(), float(t), 2,
                                     out.data_ptr(), lam.data_ptr(), self._stream), "qf_rhs")
        self._raise_errors("lambda")
        return float(lam[:, : self.n_own].max().item())

    @_on_device
    def project_initial(self) -> State:
        """Project analytic (or non-analytic ``initial``) data at t = 0 (solver.py:288-303)."""
        if self.device_setup:
            ds = self._device_initial()
            self._raise_errors("solve_velocity")
            if not self._dt_fixed:
                self.dt = cfl_time_step(self.scn.cfl, self.k, self.h_min, self.lambda_max(ds))
                ds.t_dev[1] = self.dt
                self._dt_fixed = True
            return State(t=0.0, _dev=(self, ds))
        c = self.project_fields()[: self.n_own]
        state = State(c=c, u=np.zeros((len(c), 2, self.K)), t=0.0)
        self.solve_velocity(state)
        if not self._dt_fixed and not self.partitioned:
            self.dt = self.cfl_dt(state)
            self._dt_fixed = True
        return state

    def cfl_dt(self, state: State) -> float:
        """dt = cfl * h_min / ((2k + 1) max lambda(t)) (extension)."""
        lam = self.compute_lambda(state, state.t)
        return cfl_time_step(self.scn.cfl, self.k, self.h_min, float(lam.max()))

    # --------------------------------------------------------- operators
    @_on_device
    def solve_velocity(self, state: State) -> None:
        """Per-element H-weighted projection solve, in place on state.u (solver.py:315-336)."""
        c = self._upload_c(state.c)
        _, u = self._empty_state()
        self._check(self._lib.qf_velocity(self._ctx, c.data_ptr(), u.data_ptr(), 0, -1,
                                          self._stream), "qf_velocity")
        self._raise_errors("solve_velocity")
        state.u[:] = self._soa_to_host(u, 2)

    @_on_device
    def _lam_slots(self, lam: np.ndarray):
        """Per-edge lambda in ``mesh.edges`` order -> device [3][ld] per
        (local edge, element slot), both sides of an interior edge alike."""
        lam = np.asarray(lam, dtype=np.float64)
        cn = self.mesh.conn
        if self.partitioned or lam.shape != (len(cn.left),):
            raise ValueError("lam must hold one value per mesh edge (mesh.edges order)")
        rows = np.zeros((3, self.mesh.n_triangles))
        rows[cn.left_local, cn.left] = lam
        inner = cn.right >= 0
        rows[cn.right_local[inner], cn.right[inner]] = lam[inner]
        if self.perm is not None:
            rows = rows[:, self.perm]
        out = np.zeros((3, self.ld))
        out[:, : rows.shape[1]] = rows
        return self.torch.from_numpy(out).to(self.device)

    def _rhs_terms(self, state: State, t: float, terms: int, want_lam=False, lam_in=None):
        c = self._upload_c(state.c)
        _, u = self._empty_state()
        u.zero_()
        uh = np.ascontiguousarray(state.u, dtype=np.float64)
        ua = self.torch.from_numpy(uh).to(self.device)
        self._check(self._lib.qf_pack(ua.data_ptr(), u.data_ptr(), self.tables.n_elem, 2, self.K,
                                      self.ld, self._perm_ptr(self.tables.n_elem), self._stream),
                    "qf_pack")
        out, _ = self._empty_state()
        lam = self.torch.zeros((3, self.ld), dtype=self.torch.float64, device=self.device) \
            if want_lam else None
        mass = self.instrument_mass_flux and (terms & _cabi.TERM_EDGE) and not self.partitioned
        mf = self.torch.zeros((3, self.ld), dtype=self.torch.float64, device=self.device) \
            if mass else None
        li = None if lam_in is None else self._lam_slots(lam_in)
        self._check(self._lib.qf_rhs_ex(self._ctx, c.data_ptr(), u.data_ptr(), float(t), terms,
                                        out.data_ptr(), lam.data_ptr() if want_lam else None,
                                        mf.data_ptr() if mass else None,
                                        None if li is None else li.data_ptr(), self._stream),
                    "qf_rhs_ex")
        self._raise_errors("rhs")
        r = self._soa_to_host(out, 3)
        if mass:
            self.last_mass_flux = self._mass_flux_rows(mf[:, : self.tables.n_elem].cpu().numpy())
        if want_lam:
            return r, lam[:, : self.tables.n_elem].cpu().numpy()
        return r

    def _mass_flux_rows(self, mf: np.ndarray):
        """(mL, mR) over the interior edges in mesh.edges order (reference
        solver.py:696-701): the element's mass rate sqrt(detB)/sqrt(2) *
        (xi mode-0 rhs) through the edge, for its left / right element."""
        if self.perm is not None:
            rows = np.empty_like(mf)
            rows[:, self.perm] = mf
            mf = rows
        mf = mf * (self.geom.sqrt_detB / math.sqrt(2.0))[None, :]
        cn = self.mesh.conn
        inner = np.flatnonzero(cn.right >= 0)
        return (mf[cn.left_local[inner], cn.left[inner]],
                mf[cn.right_local[inner], cn.right[inner]])

    def compute_lambda(self, state: State, t: float) -> np.ndarray:
        """Per-edge LF speed in ``mesh.edges`` order (solver.py:340-406)."""
        if self.partitioned:
            raise NotImplementedError("compute_lambda on a partition: use lambda_local")
        _, lam = self._rhs_terms(state, t, _cabi.TERM_EDGE, want_lam=True)
        if self.perm is not None:
            lam_rows = np.empty_like(lam)
            lam_rows[:, self.perm] = lam
            lam = lam_rows
        c = self.mesh.conn
        return lam[c.left_local, c.left]

    def element_rhs(self, state: State) -> np.ndarray:
        return self._rhs_terms(state, 0.0, _cabi.TERM_VOLUME)

    def edge_rhs(self, state: State, t: float, lam: np.ndarray | None = None) -> np.ndarray:
        """Edge terms (solver.py:690-706); a given ``lam`` (per edge, mesh.edges
        order, as compute_lambda returns it) is used in the Lax-Friedrichs
        flux instead of the recomputed one, like the reference."""
        return self._rhs_terms(state, t, _cabi.TERM_EDGE, lam_in=lam)

    def source_rhs(self, state: State, t: float) -> np.ndarray:
        return self._rhs_terms(state, t, _cabi.TERM_SOURCE)

    def rhs(self, state: State, t: float) -> np.ndarray:
        r, lam = self._rhs_terms(state, t, _cabi.TERM_ALL, want_lam=True)
        self._cfl_advisory(float(lam.max()))
        return r

    def _cfl_advisory(self, lam_max: float):
        if not self._cfl_warned:
            cfl = self.dt * lam_max / self.h_min
            if cfl > self.cfl_warn_threshold:
                warnings.warn(f"CFL advisory: dt*lambda_max/h_min = {cfl:.2f} exceeds "
                              f"{self.cfl_warn_threshold}", stacklevel=3)
            self._cfl_warned = True

    # ------------------------------------------------------ time stepping
    @_on_device
    def l2_error_sq(self, state, t: float) -> np.ndarray:
        """Squared L2 errors (xi, U, V) of the owned elements against the
        scenario's exact solution at t, evaluated on the device (qf_l2_error;
        reference harness.py:81-98).  ``state``: State or DeviceState."""
        ds = state if isinstance(state, DeviceState) else self.to_device(state, solve=False)
        sq = self.torch.zeros(3, dtype=self.torch.float64, device=self.device)
        self._check(self._lib.qf_l2_error(self._ctx, ds.c.data_ptr(), float(t), 0, self.n_own,
                                          sq.data_ptr(), self._stream), "qf_l2_error")
        return sq.cpu().numpy()

    def _work_buf(self):
        if self._work is None:
            self._work = self.torch.empty(2 * 5 * self.K * self.ld, dtype=self.torch.float64,
                                          device=self.device)
        return self._work

    @_on_device
    def step_device(self, ds: DeviceState, n_steps: int = 1, use_graph: bool = True) -> None:
        """Advance a device state in place by n_steps (no host traffic)."""
        w = self._work_buf()
        if n_steps == 1:
            st = self._lib.qf_step(self._ctx, ds.c.data_ptr(), ds.u.data_ptr(), w.data_ptr(),
                                   ds.t_dev.data_ptr(), self._stream)
            self._check(st, "qf_step")
        elif n_steps > 1:
            st = self._lib.qf_run(self._ctx, n_steps, ds.c.data_ptr(), ds.u.data_ptr(),
                                  w.data_ptr(), ds.t_dev.data_ptr(), 1 if use_graph else 0,
                                  self._stream)
            self._check(st, "qf_run")

    @_on_device
    def step(self, state: State) -> State:
        """One SSP-RK step; returns a new State, input unchanged (solver.py:745-770)."""
        ds = self.to_device(state).clone() if state._dev is not None else self.to_device(state)
        ds.t_dev[1] = self.dt
        if not self._cfl_warned:
            self._cfl_advisory(float(self.compute_lambda(State(t=state.t, _dev=(self, ds.clone())),
                                                         state.t).max()))
        self.step_device(ds, 1)
        self._raise_errors(f"step to t = {state.t + self.dt}")
        return State(t=state.t + self.dt, _dev=(self, ds))

    @_on_device
    def run(self, state: State | None = None, t_end: float | None = None) -> State:
        if state is None:
            state = self.project_initial()
        t_end = self.scn.t_end if t_end is None else t_end
        n_steps = int(round((t_end - state.t) / self.dt))
        ds = self.to_device(state)
        if state._dev is not None:
            ds = ds.clone()
        ds.t_dev[1] = self.dt
        self.step_device(ds, n_steps)
        self._raise_errors(f"run to t = {t_end}")
        t = float(ds.t_dev[0].item())
        return State(t=t, _dev=(self, ds))
