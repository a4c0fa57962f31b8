"""GPU parity pinned to the reference at the BASELINE configs' stated step
counts (reduced N), plus the p = 4 convergence orders and the SPEC flux
consistency invariant.  Tolerance: 1e-11 relative L2 per field.

Fixtures (tests/golden/make_golden.py --walls, run against the reference):
* walls_p3_n16 -- C3 physics (bumps at rest, seeded sine bathymetry,
  reflective walls, CFL dt), p = 3, N = 16, 500 SSP-RK3 steps;
* walls_p2_j16 -- C4 physics on the 0.2 h jittered mesh, p = 2, N = 16, 300 steps;
* mms_p2_n16   -- C2 schedule (MMS, SSP-RK3, dt = 2e-5), p = 2, N = 16, 1000 steps.
The reference runs through a documented subclass (mirror-ghost
``_boundary_flux``, wall branch of ``compute_lambda``); N = 16 puts four
128-element Morton blocks on the mesh, so in-block and out-of-block
neighbour traces are both exercised.
"""

import numpy as np
import pytest

from conftest import field_rel, rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.mark.parametrize("name,k,jitter", [("walls_p3_n16", 3, 0.0), ("walls_p2_j16", 2, 0.2)])
def test_walls_bumps_vs_reference_stated_steps(golden, name, k, jitter):
    from paper_1904_08684_b200 import mesh as M, scenario as S
    from paper_1904_08684_b200.solver import Discretization
    g = golden(f"{name}.npz")
    mesh = M.build_unit_square_mesh(16, jitter=jitter, seed=7)
    assert np.array_equal(mesh.vertices, g["verts"])  # same generator bits as the fixture
    scn = S.bump_scenario(seed=0, cfl=0.1)
    assert scn.name == f"bumps-seed{int(g['seed'])}"
    disc = Discretization(mesh, scn, k)
    st0 = disc.project_initial()
    assert field_rel(st0.c, g["c0"]) < TOL
    assert field_rel(st0.u, g["u0"]) < TOL
    # CFL convention: dt = 0.1 h_min / ((2k + 1) lambda_max(0)), h_min and
    # lambda as the reference computes them
    assert abs(disc.h_min - float(g["h_min"])) <= 1e-15 * float(g["h_min"])
    assert abs(disc.dt - float(g["dt"])) <= 1e-13 * float(g["dt"])
    assert rel_l2(disc.compute_lambda(st0, 0.0), g["lam"]) < TOL
    assert field_rel(disc.element_rhs(st0), g["elem"]) < TOL
    assert field_rel(disc.edge_rhs(st0, 0.0), g["edge"]) < TOL
    assert field_rel(disc.source_rhs(st0, 0.0), g["src"]) < TOL
    assert field_rel(disc.rhs(st0, 0.0), g["rhs0"]) < TOL
    st = disc.step(st0)
    assert field_rel(st.c, g["c1"]) < TOL
    st = disc.run(st, t_end=10 * disc.dt)
    assert field_rel(st.c, g["c10"]) < TOL
    steps = int(g["steps"])
    out = disc.run(st, t_end=steps * disc.dt)
    assert abs(out.t - steps * disc.dt) < 1e-12
    for j in range(3):  # per field, after the stated step count
        assert rel_l2(out.c[:, j], g["cN"][:, j]) < TOL
    assert field_rel(out.u, g["uN"]) < TOL


def test_c2_schedule_1000_steps_vs_reference(golden):
    """C2 schedule in full (1000 SSP-RK3 steps, dt = 2e-5) at N = 16."""
    from paper_1904_08684_b200 import harness as Hn, mesh as M, scenario as S
    from paper_1904_08684_b200.solver import Discretization
    g = golden("mms_p2_n16.npz")
    disc = Discretization(M.build_unit_square_mesh(16), S.mms_scenario(dt=2e-5, t_end=0.02), 2)
    st0 = disc.project_initial()
    assert field_rel(st0.c, g["c0"]) < TOL
    out = disc.run(st0)
    assert abs(out.t - float(g["t"])) < 1e-12
    for j in range(3):
        assert rel_l2(out.c[:, j], g["cN"][:, j]) < TOL
    assert field_rel(out.u, g["uN"]) < TOL
    err = Hn.l2_error(disc, out, out.t).errors()
    assert np.allclose(err, g["err"], rtol=1e-9, atol=0)


def p4_sweep(hb, ns):
    from paper_1904_08684_b200 import harness as Hn, mesh as M, scenario as S
    scn = S.mms_scenario(dt=2e-5, t_end=0.02, hb_coeffs=hb)
    return Hn.convergence_study(4, ns, scenario=scn,
                                mesh_builder=lambda n: M.build_unit_square_mesh(int(n)))


HB_LINEAR, HB_BILINEAR = (1.0, 0.1, 0.05, 0.0), (1.0, 0.0, 0.0, 0.1)


def test_p4_convergence_linear_bathymetry(golden):
    """p = 4 MMS (C2 schedule: SSP-RK3, dt = 2e-5, 1000 steps) over a linear
    h_b (P1 projection exact): design order k + 1 = 5; errors at the
    overlapping N equal the CPU oracle's p = 4 extension
    (tests/golden/sweep_p4_oracle.npz, make_sweep_p4.py)."""
    g = golden("sweep_p4_oracle.npz")
    ns = [4, 8, 16, 32, 64]
    tab = p4_sweep(HB_LINEAR, ns)
    err = np.array([r.errors() for r in tab.rows])
    print(tab.to_csv())
    assert np.allclose(err[:len(g["n"])], g["err_linear"], rtol=1e-9, atol=0)
    eoc = np.array(tab.eoc())
    # measured (B200): EOC(xi) 5.02 5.01 5.01 5.00; EOC(U, V) 4.83 5.03 4.91 4.76
    # (U, V at N = 64 reach 3e-11, where the SSP-RK3 time error starts to show)
    assert (eoc[:, 0] > 4.9).all(), eoc
    assert (eoc[:, 1:] > 4.7).all(), eoc


def test_p4_bathymetry_bilinear_matches_oracle(golden):
    """p = 4 with the BASELINE bilinear h_b: errors equal the oracle's (the
    P1 projection of h_b caps the order, as SURVEY App. C shows for p = 3)."""
    g = golden("sweep_p4_oracle.npz")
    tab = p4_sweep(HB_BILINEAR, list(g["n"]))
    err = np.array([r.errors() for r in tab.rows])
    assert np.allclose(err, g["err_bilinear"], rtol=1e-9, atol=0)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_flux_consistency_identical_traces(k):
    """SPEC.md invariant (flux consistency): with identical traces on both
    sides of every interior edge (globally continuous polynomial fields of
    degree <= k), the Lax-Friedrichs edge term equals the analytic
    flux_dot_n (reference solver.py:60-71) integrated by an independent
    pointwise oracle at 5 Gauss points per edge, to 1e-12."""
    from paper_1904_08684_b200 import mesh as M, scenario as S
    from paper_1904_08684_b200.solver import Discretization, State, flux_dot_n
    mesh = M.build_unit_square_mesh(6, jitter=0.2, seed=11)
    hb = lambda x, y: 1.5 + 0.1 * np.asarray(x) - 0.2 * np.asarray(y)  # noqa: E731
    scn = S.Scenario(name="poly", dt=1e-3, dirichlet_markers=frozenset(),
                     wall_markers=frozenset({1}), hb=hb)
    disc = Discretization(mesh, scn, k)
    rng = np.random.default_rng(k)
    P = rng.standard_normal((5, k + 1, k + 1)) * 0.05

    def field(f):  # global polynomial of degree <= k
        def fn(x, y):
            x, y = np.asarray(x), np.asarray(y)
            return sum(P[f, a, b] * x**a * y**b for a in range(k + 1) for b in range(k + 1 - a))
        return fn

    fl = [field(f) for f in range(5)]
    fl[0] = (lambda f0: (lambda x, y: 0.3 + f0(x, y)))(fl[0])
    c = np.stack([disc.project_volume(fl[f]) for f in range(3)], axis=1)
    u = np.stack([disc.project_volume(fl[f]) for f in (3, 4)], axis=1)
    got = disc.edge_rhs(State(c, u, 0.0), 0.0)
    # independent pointwise oracle
    # (SPEC: 5 points; the edge integrand phi_p * flux has degree 3k, so
    # k = 4 needs 7 for an exact oracle: use 8 everywhere)
    s, w = np.polynomial.legendre.leggauss(8)
    s, w = 0.5 * (s + 1.0), 0.5 * w
    geo = disc.geom
    cn = mesh.conn
    has_bnd = np.zeros(mesh.n_triangles, bool)
    has_bnd[cn.left[cn.right < 0]] = True
    want = np.zeros_like(got)
    basis = disc.basis.functions
    ends = (((1.0, 0.0), (0.0, 1.0)), ((0.0, 1.0), (0.0, 0.0)), ((0.0, 0.0), (1.0, 0.0)))
    for e in np.flatnonzero(~has_bnd):
        B, a1, sd = geo.B[e], geo.a1[e], geo.sqrt_detB[e]
        for (r0, r1) in ends:
            r0, r1 = np.array(r0), np.array(r1)
            d = B @ (r1 - r0)
            ln = np.hypot(*d)
            n1, n2 = d[1] / ln, -d[0] / ln
            for sg, wg in zip(s, w):
                r = r0 + sg * (r1 - r0)
                x, y = a1 + B @ r
                vals = [fl[f](x, y) for f in range(5)]
                F = flux_dot_n(vals[0], vals[1], vals[2], vals[3], vals[4], hb(x, y), n1, n2,
                               scn.g)
                phi = np.array([f.eval_point(r[0], r[1]) for f in basis]) / sd
                for q in range(3):
                    want[e, q] -= ln * wg * F[q] * phi
    sel = ~has_bnd
    scale = np.abs(want[sel]).max()
    assert np.abs(got[sel] - want[sel]).max() <= 1e-12 * scale


@pytest.mark.parametrize("k", [1, 2, 3])
def test_edge_rhs_uses_given_lambda(golden, k):
    """edge_rhs(state, t, lam) uses the caller's lambda in the LF flux like the
    reference (solver.py:690-704): a scaled lambda changes the result exactly
    as it does in the oracle, and lam = compute_lambda reproduces the default."""
    from oracle import qfswe_oracle as O
    from paper_1904_08684_b200 import mesh as M, scenario as S
    from paper_1904_08684_b200.solver import Discretization, State
    g = golden(f"square_k{k}.npz")
    mesh = M.build_square_mesh(3, 0.2, 42)
    disc = Discretization(mesh, S.perturbed_square_scenario(dt=0.5), k)
    st = State(g["cr"].copy(), g["ur"].copy(), 0.0)
    lam = disc.compute_lambda(st, 3.7)
    assert np.array_equal(disc.edge_rhs(st, 3.7, lam), disc.edge_rhs(st, 3.7))
    orc = O.OracleSolver(O.OMesh(mesh.vertices, mesh.triangles), O.travel_wave(dt=0.5), k)
    olam = orc.compute_lambda(g["cr"], g["ur"], 3.7)
    want = orc.edge_rhs(g["cr"], g["ur"], 3.7, lam=1.5 * olam)
    assert field_rel(disc.edge_rhs(st, 3.7, 1.5 * lam), want) < TOL


@pytest.mark.parametrize("k", [1, 2, 3])
def test_custom_scenario_on_device_vs_reference(golden, k):
    """A reference ``custom_scenario`` with Dirichlet data and manufactured
    forcing runs on the B200 path: its SymPy fields are compiled into a
    per-scenario device module (csrc/qf_user.cuh, qf_user_scenario) that
    the stage / ghost launches use every stage; terms and 5 steps equal the
    reference's (tests/golden/custom_k*.npz, make_golden.py --custom)."""
    import sys
    from paper_1904_08684_b200 import mesh as M, scenario as S
    from paper_1904_08684_b200.solver import Discretization, State
    sys.path.insert(0, __file__.rsplit("/", 1)[0] + "/golden")
    from make_golden import CUSTOM_FIELDS
    g = golden(f"custom_k{k}.npz")
    scn = S.custom_scenario(*CUSTOM_FIELDS, dt=0.5)
    assert scn.device.kind == S.KIND_USER and scn.forcing is not None
    disc = Discretization(M.build_square_mesh(3, 0.2, 42), scn, k)
    st0 = disc.project_initial()
    assert field_rel(st0.c, g["c0"]) < TOL
    sr = State(g["cr"].copy(), g["ur"].copy(), 0.0)
    assert rel_l2(disc.compute_lambda(sr, 2.3), g["lam"]) < TOL
    assert field_rel(disc.edge_rhs(sr, 2.3), g["edge"]) < TOL
    assert field_rel(disc.source_rhs(sr, 2.3), g["src"]) < TOL
    assert field_rel(disc.rhs(sr, 2.3), g["rhs_r"]) < TOL
    out = disc.run(st0, t_end=2.5)
    assert field_rel(out.c, g["c5"]) < TOL
    assert field_rel(out.u, g["u5"]) < TOL


def test_family_scenario_edited_after_construction_is_rejected():
    """ADVICE: the kernels evaluate a closed-form family; a scenario whose
    callables were replaced afterwards would run mixed physics, so it is
    refused (dataclasses.replace of unrelated fields is fine)."""
    import dataclasses
    from paper_1904_08684_b200 import mesh as M, scenario as S
    from paper_1904_08684_b200.solver import Discretization
    mesh = M.build_unit_square_mesh(4)
    scn = S.mms_scenario(dt=1e-4)
    Discretization(mesh, dataclasses.replace(scn, dt=2e-4), 1)
    bad = S.mms_scenario(dt=1e-4)
    bad.exact = lambda x, y, t: (x * 0, x * 0, x * 0)
    with pytest.raises(ValueError):
        Discretization(mesh, bad, 1)
    with pytest.raises(ValueError):
        Discretization(mesh, dataclasses.replace(scn, g=1.0), 1)


@pytest.mark.parametrize("case", ["unit_walls", "jitter_mms", "square_travel", "ragged"])
def test_device_tables_equal_host_tables(case):
    """Device-side setup (device_setup.py: connectivity by a device sort,
    geometry, Z-order slots, SoA tables) reproduces the host NumPy setup
    (mesh.build_connectivity / compute_geometry / locality_order /
    layout.build_tables) bit for bit."""
    from paper_1904_08684_b200 import mesh as M, scenario as S
    from paper_1904_08684_b200.device_setup import device_tables
    from paper_1904_08684_b200.solver import HostSetup
    mesh, scn = {
        "unit_walls": (M.build_unit_square_mesh(48), S.bump_scenario(seed=0, cfl=0.1)),
        "jitter_mms": (M.build_unit_square_mesh(40, jitter=0.2, seed=7), S.mms_scenario(dt=1e-4)),
        "square_travel": (M.build_square_mesh(5, 0.2, 42), S.perturbed_square_scenario(dt=0.5)),
        "ragged": (M.build_unit_square_mesh(13), S.mms_scenario(dt=1e-4)),
    }[case]
    host = HostSetup(mesh, scn, 2, device_tables=False).tables
    dev = device_tables(mesh, scn.dirichlet_markers, scn.wall_markers, "cuda")
    perm = HostSetup(mesh, scn, 2, device_tables=False).perm
    assert np.array_equal(dev.host("perm"), perm)
    assert np.array_equal(dev.host("geo"), host.geo)
    assert np.array_equal(dev.host("nbr"), host.nbr)
    assert np.array_equal(dev.host("bnd_elem"), host.bnd_elem)
    assert np.array_equal(dev.host("bnd_local"), host.bnd_local)
    assert dev.h_min == host.h_min and dev.ld == host.ld and dev.n_elem == host.n_elem


def test_device_tables_run_matches_host_setup():
    """A whole run on device-built tables equals the host-built one exactly."""
    from paper_1904_08684_b200 import mesh as M, scenario as S
    from paper_1904_08684_b200.solver import Discretization
    mesh = M.build_unit_square_mesh(32, jitter=0.2, seed=7)
    scn = S.bump_scenario(seed=0, cfl=0.1)
    a = Discretization(mesh, scn, 3, device_setup=True, device_tables=False)
    b = Discretization(mesh, scn, 3, device_setup=True, device_tables=True)
    assert b.device_tables and not a.device_tables
    ra = a.run(a.project_initial(), t_end=5 * a.dt)
    rb = b.run(b.project_initial(), t_end=5 * b.dt)
    assert a.dt == b.dt
    assert np.array_equal(ra.c, rb.c) and np.array_equal(ra.u, rb.u)
