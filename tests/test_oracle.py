"""CPU: the oracle (test infrastructure) pinned against reference fixtures,
and the reformulated trace-space algorithm against the dense oracle."""

import numpy as np
import pytest

from conftest import field_rel, rel_l2

from oracle import qfswe_oracle as O
from oracle import trace_stage as TS
from paper_1904_08684_b200 import layout as L
from paper_1904_08684_b200 import mesh as M
from paper_1904_08684_b200 import scenario as S


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_oracle_tensors_vs_reference(golden, k):
    t = O.build_tensors(k)
    g = golden(f"tensors_k{k}.npz")
    for name in g.files:
        ref = g[name]
        assert np.abs(getattr(t, name) - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), name


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_oracle_square_vs_reference(golden, k):
    g = golden(f"square_k{k}.npz")
    m = M.build_square_mesh(3, 0.2, 42)
    s = O.OracleSolver(O.OMesh(m.vertices, m.triangles), O.travel_wave(dt=0.5), k)
    c0, u0 = s.project_initial()
    assert field_rel(c0, g["c0"]) < 1e-13
    cr, ur = g["cr"], g["ur"]
    assert field_rel(s.solve_velocity(cr), ur) < 1e-13
    assert rel_l2(s.compute_lambda(cr, ur, 3.7), g["lam"]) < 1e-13
    assert field_rel(s.element_rhs(cr, ur), g["elem"]) < 1e-13
    assert field_rel(s.edge_rhs(cr, ur, 3.7), g["edge"]) < 1e-13
    assert field_rel(s.source_rhs(cr, 3.7), g["src"]) < 1e-13
    c3, u3, _ = s.run(g["c0"], 0.0, 3)
    assert field_rel(c3, g["c3"]) < 1e-12


def test_oracle_c1_terms_vs_reference(golden):
    g = golden("c1_mms_p1_n32.npz")
    m = M.build_unit_square_mesh(32)
    s = O.OracleSolver(O.OMesh(m.vertices, m.triangles), O.mms_baseline(dt=1e-4), 1)
    c0, u0 = s.project_initial()
    assert field_rel(c0, g["c0"]) < 1e-13
    assert rel_l2(s.compute_lambda(c0, u0, 0.0), g["lam"]) < 1e-13
    assert field_rel(s.edge_rhs(c0, u0, 0.0), g["edge"]) < 1e-13
    assert field_rel(s.source_rhs(c0, 0.0), g["src"]) < 1e-13
    c, _, _ = s.run(c0, 0.0, 20)  # full 200-step run is covered on the GPU


@pytest.mark.slow
def test_oracle_c1_full_vs_reference(golden):
    g = golden("c1_mms_p1_n32.npz")
    m = M.build_unit_square_mesh(32)
    s = O.OracleSolver(O.OMesh(m.vertices, m.triangles), O.mms_baseline(dt=1e-4), 1)
    c0, _ = s.project_initial()
    c, _, t = s.run(c0, 0.0, 200)
    assert field_rel(c, g["c200"]) < 1e-12
    assert np.allclose(s.l2_error(c, t), g["err"], rtol=1e-9)


@pytest.mark.parametrize("k,n", [(2, 8), (3, 6)])
def test_oracle_mms_vs_reference(golden, k, n):
    g = golden(f"mms_p{k}_n{n}.npz")
    m = M.build_unit_square_mesh(n)
    s = O.OracleSolver(O.OMesh(m.vertices, m.triangles), O.mms_baseline(dt=2e-5), k)
    c0, _ = s.project_initial()
    assert field_rel(c0, g["c0"]) < 1e-13
    assert field_rel(s.edge_rhs(g["cr"], g["ur"], 0.3), g["edge"]) < 1e-13
    cN, _, _ = s.run(c0, 0.0, int(g["steps"]))
    assert field_rel(cN, g["cN"]) < 1e-12


def test_oracle_ring_and_lake(golden):
    g = golden("ring_k1.npz")
    m = M.build_ring_mesh(2)
    s = O.OracleSolver(O.OMesh(m.vertices, m.triangles), O.travel_wave(dt=0.5), 1)
    c0, _ = s.project_initial()
    c2, _, _ = s.run(c0, 0.0, 2)
    assert field_rel(c2, g["c2"]) < 1e-12
    for k in (1, 2, 3):
        g = golden(f"lake_k{k}.npz")
        m = M.build_square_mesh(2, 0.2, 5)
        s = O.OracleSolver(O.OMesh(m.vertices, m.triangles), O.lake(dt=0.5), k)
        c0, u0 = s.project_initial()
        assert np.abs(s.rhs(c0, u0, 0.0)).max() < 1e-10
        c10, _, _ = s.run(c0, 0.0, 10)
        assert np.abs(c10 - g["c10"]).max() < 1e-12


def _trace_setup(m, oscn, pscn, k):
    ors = O.OracleSolver(O.OMesh(m.vertices, m.triangles), oscn, k)
    tb = L.build_tables(m, oscn.dirichlet_markers, oscn.wall_markers)
    nh = 1 if k == 0 else 3
    hb = np.zeros((nh, tb.ld))
    hb[:, : m.n_triangles] = ors.hb[:, :nh].T
    ts = TS.TraceStage(k, tb.geo, tb.nbr, hb, m.n_triangles, pscn, tb.bnd_elem, tb.bnd_local)
    return ors, ts, tb


@pytest.mark.parametrize("case,k", [("square", 1), ("square", 3), ("mms", 0), ("mms", 2),
                                    ("mms", 4), ("walls", 2), ("walls", 4)])
def test_trace_space_reformulation_vs_dense(case, k):
    """The kernel algorithm (trace-space edges, factorised volume) == dense oracle."""
    if case == "square":
        m = M.build_square_mesh(3, 0.2, 42)
        oscn, pscn = O.travel_wave(dt=0.5), S.perturbed_square_scenario(dt=0.5)
        noise = 0.05
    elif case == "mms":
        m = M.build_unit_square_mesh(6)
        oscn, pscn = O.mms_baseline(dt=1e-4), S.mms_scenario(dt=1e-4)
        noise = 0.05
    else:
        m = M.build_unit_square_mesh(16)
        pscn = S.bump_scenario(seed=0, dt=1e-3)
        oscn = O.OScenario(dt=1e-3, dirichlet_markers=frozenset(), wall_markers=frozenset({1}),
                           hb=pscn.hb, initial=pscn.initial)
        noise = 0.0
    ors, ts, tb = _trace_setup(m, oscn, pscn, k)
    c0, _ = ors.project_initial()
    rng = np.random.default_rng(3)
    cr = c0 * (1 + noise * rng.standard_normal(c0.shape)) if noise else \
        c0 + 1e-5 * rng.standard_normal(c0.shape)
    ur = ors.solve_velocity(cr)
    E = m.n_triangles
    cs, us = L.aos_to_soa(cr, tb.ld), L.aos_to_soa(ur, tb.ld)

    def aos(x):
        return np.ascontiguousarray(x.transpose(2, 0, 1))[:E]

    assert field_rel(aos(ts.velocity(cs)), ur) < 1e-12
    lam = np.zeros((3, tb.ld))
    for terms, ref in ((1, ors.element_rhs(cr, ur)), (2, ors.edge_rhs(cr, ur, 0.3)),
                       (4, ors.source_rhs(cr, 0.3))):
        assert field_rel(aos(ts.rhs(cs, us, 0.3, terms, lam)), ref) < 1e-12
    lref = ors.compute_lambda(cr, ur, 0.3)
    assert np.abs(lam[:, :E].T - lref[m.conn.elem_edge]).max() <= 1e-13 * lref.max()
