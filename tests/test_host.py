"""CPU: host setup (exact basis/tensors, mesh, layout, scenarios, codegen)
and the C-ABI library surface (loads and exports; no compute calls)."""

import math
import os
import re
from fractions import Fraction

import numpy as np
import pytest

from conftest import ROOT
from paper_1904_08684_b200 import layout as L
from paper_1904_08684_b200 import mesh as M
from paper_1904_08684_b200 import scenario as S
from paper_1904_08684_b200 import symbolic as SY
from paper_1904_08684_b200 import tensors as T

REF = "/root/reference/pkg/src/qfswe"
needs_ref = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


def _ref():
    import importlib
    import sys
    import types
    if "qfswe_ref" not in sys.modules:
        pkg = types.ModuleType("qfswe_ref")
        pkg.__path__ = [REF]
        sys.modules["qfswe_ref"] = pkg
    return importlib.import_module("qfswe_ref.mesh")


# ------------------------------------------------------------ symbolic
def test_spec_known_answers():
    assert SY.monomial_integral(0, 0) == Fraction(1, 2)
    assert SY.monomial_integral(1, 0) == Fraction(1, 6)
    assert SY.monomial_integral(1, 1) == Fraction(1, 24)
    t = T.build_ref_tensors(1)
    assert t.S[0, 1, 0] == -3 * math.sqrt(2)
    assert abs(t.G[0, 0, 0] - math.sqrt(2)) < 1e-15


@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_exact_orthonormality(k):
    b = SY.build_basis(k)
    for p, fp in enumerate(b.functions):
        for i, fi in enumerate(b.functions):
            r, m = (fp * fi).integral()
            assert m == 1 and r == (1 if p == i else 0)


def test_p4_extension_is_hierarchical():
    b3, b4 = SY.build_basis(3), SY.build_basis(4)
    assert b4.functions[:10] == b3.functions
    assert all(f.degree == 4 for f in b4.functions[10:])


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_tensors_bit_identical_to_reference(golden, k):
    t = T.build_ref_tensors(k)
    g = golden(f"tensors_k{k}.npz")
    for name in g.files:
        assert np.array_equal(t.as_dict()[name], g[name]), name


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_tensor_csv_dump_byte_identical_to_reference(golden, tmp_path, k):
    """dump_tensors_csv writes the reference's files byte for byte
    (reference tensors.py:257-275); load_tensors_csv inverts it."""
    import hashlib
    g = golden("tensor_files.npz")
    t = T.build_ref_tensors(k)
    for path in T.dump_tensors_csv(t, tmp_path):
        assert hashlib.sha256(path.read_bytes()).hexdigest() == str(g[f"sha_{path.stem}"]), path.name
    back = T.load_tensors_csv(k, tmp_path)
    for name, x in t.as_dict().items():
        assert np.array_equal(x, back.as_dict()[name]), name


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_verify_tensors_report(golden, k):
    """verify_tensors (reference tensors.py:207-254): frozen vs quadrature at
    roundoff, same magnitude as the reference's own report."""
    rep = T.verify_tensors(T.build_ref_tensors(k))
    assert rep.order == k and rep.max_rel_dev < 1e-13
    if k <= 3:
        ref_abs, ref_rel = golden("tensor_files.npz")[f"report_k{k}"]
        assert rep.max_abs_dev < 10 * ref_abs + 1e-15 and rep.max_rel_dev < 10 * ref_rel + 1e-16


def test_p4_tensors_vs_quadrature():
    from oracle import qfswe_oracle as O
    a, b = T.build_ref_tensors(4), O.build_tensors(4)
    assert np.array_equal(a.M, np.eye(15))
    for name, x in a.as_dict().items():
        y = getattr(b, name)
        assert np.abs(x - y).max() <= 1e-11 * np.abs(y).max(), name


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_trace_space_identities(k):
    t, ts = T.build_ref_tensors(k), T.build_trace_space(k)
    R = (-1.0) ** np.arange(k + 1)
    tol = 1e-13 * np.abs(t.ETX).max()
    assert np.abs(np.einsum("eia,eja->eij", ts.Lam, ts.Lam) - t.E).max() < tol
    assert np.abs(np.einsum("eia,fja,a->efij", ts.Lam, ts.Lam, R) - t.EX).max() < tol
    ET = np.einsum("epa,eib,emc,abc->epim", ts.Lam, ts.Lam, ts.Lam, ts.J)
    ETX = np.einsum("epa,fib,fmc,abc,b,c->efpim", ts.Lam, ts.Lam, ts.Lam, ts.J, R, R)
    assert np.abs(ET - t.ET).max() < tol
    assert np.abs(ETX - t.ETX).max() < tol


def test_quadrature_rules_match_reference_construction():
    p, w = T.triangle_rule(6)
    assert len(w) == 16 and abs(w.sum() - 0.5) < 1e-15
    s, w1 = T.edge_rule(7)
    assert len(s) == 4 and abs(w1.sum() - 1.0) < 1e-15


# ---------------------------------------------------------------- mesh
@needs_ref
@pytest.mark.parametrize("lv,pert,seed", [(2, 0.2, 42), (3, 0.2, 7), (4, 0.0, 0)])
def test_square_mesh_identical_to_reference(lv, pert, seed):
    R = _ref()
    a, b = M.build_square_mesh(lv, pert, seed), R.build_square_mesh(lv, pert, seed)
    assert np.array_equal(a.vertices, b.vertices) and np.array_equal(a.triangles, b.triangles)
    key = lambda e: (e.v0, e.v1, e.left, e.left_local, e.right, e.right_local, e.marker)  # noqa
    assert [key(e) for e in a.edges] == [key(e) for e in b.edges]
    ga, ea = M.compute_geometry(a)
    gb, eb = R.compute_geometry(b)
    assert np.array_equal(ga.B, gb.B) and np.array_equal(ea.normal, eb.normal)


@needs_ref
def test_ring_mesh_identical_to_reference():
    R = _ref()
    a, b = M.build_ring_mesh(2), R.build_ring_mesh(2)
    assert np.array_equal(a.triangles, b.triangles)
    assert np.abs(a.vertices - b.vertices).max() == 0.0


@pytest.mark.parametrize("n", [1, 4, 32])
def test_unit_square_counts(n):
    m = M.build_unit_square_mesh(n)
    c = m.conn
    assert m.n_triangles == 2 * n * n
    assert c.n_edges == 3 * n * n + 2 * n
    assert int((c.right < 0).sum()) == 4 * n
    g, _ = M.compute_geometry(m)
    assert np.allclose(g.detB, 1.0 / n**2)


def test_jitter_interior_only_and_valid():
    m0, m1 = M.build_unit_square_mesh(16), M.build_unit_square_mesh(16, 0.2, 9)
    d = np.abs(m1.vertices - m0.vertices).max(axis=1)
    x, y = m0.vertices[:, 0], m0.vertices[:, 1]
    bnd = (x == 0) | (x == 1) | (y == 0) | (y == 1)
    assert (d[bnd] == 0).all() and (d[~bnd] > 0).all() and d.max() <= 0.2 / 16
    assert (M.compute_geometry(m1)[0].detB > 0).all()
    assert np.array_equal(M.build_unit_square_mesh(16, 0.2, 9).vertices, m1.vertices)


def test_connectivity_errors(tmp_path):
    v = np.array([[0, 0], [1, 0], [0, 1], [1, 1]], dtype=float)
    with pytest.raises(M.ConnectivityError):
        M._finish(v, np.array([[0, 1, 2], [0, 1, 2]]))
    with pytest.raises(M.ConnectivityError):
        M._finish(np.vstack([v, [[0.5, -1]]]), np.array([[0, 1, 2], [1, 3, 2], [0, 4, 1], [1, 0, 4]]))
    m = M.build_square_mesh(2, 0.1, 3)
    p = tmp_path / "m.txt"
    M.save_mesh(m, p)
    m2 = M.load_mesh(p)
    assert np.array_equal(m2.vertices, m.vertices) and np.array_equal(m2.triangles, m.triangles)
    p.write_text("ghoddess-mesh 1\nvertices 1\n0 0 0\n")
    with pytest.raises(M.MeshParseError, match="line 3"):
        M.load_mesh(p)


def test_layout_tables_are_consistent():
    m = M.build_square_mesh(3, 0.2, 1)
    tb = L.build_tables(m, frozenset({1}), frozenset())
    E = m.n_triangles
    code = tb.nbr[:, :E].astype(np.int64)
    for j in range(3):
        inner = code[j] >= 0
        e = np.flatnonzero(inner)
        nb, jn = code[j, inner] >> 2, code[j, inner] & 3
        back = code[jn, nb]
        assert np.array_equal(back >> 2, e) and np.array_equal(back & 3, np.full_like(e, j))
    # Dirichlet slots follow the reference's pass_B (mesh-edge) order
    c = m.conn
    bidx = np.flatnonzero(c.right < 0)
    assert np.array_equal(tb.bnd_elem, c.left[bidx]) and np.array_equal(tb.bnd_local, c.left_local[bidx])
    with pytest.raises(ValueError):
        L.build_tables(m, frozenset({7}), frozenset())


def test_aos_soa_roundtrip():
    a = np.random.default_rng(0).standard_normal((37, 3, 6))
    s = L.aos_to_soa(a, L.pad_ld(37))
    assert s.shape == (3, 6, 64) and np.array_equal(L.soa_to_aos(s, 37), a)


# ------------------------------------------------------------ scenarios
def test_mms_forcing_matches_sympy():
    import sympy as sp
    X, Y, Tt = sp.symbols("x y t", real=True)
    xi = sp.sin(2 * sp.pi * (X + Y - Tt)) / 100
    hb = 1 + X * Y / 10
    H = hb + xi
    U = H * sp.cos(2 * sp.pi * (X - Tt)) / 10
    V = H * sp.sin(2 * sp.pi * (Y - Tt)) / 10
    g = sp.Float(9.81)
    ex = [sp.diff(U, Tt) + sp.diff(U**2 / H, X) + sp.diff(U * V / H, Y) + g * H * sp.diff(xi, X),
          sp.diff(V, Tt) + sp.diff(U * V / H, X) + sp.diff(V**2 / H, Y) + g * H * sp.diff(xi, Y),
          sp.diff(xi, Tt) + sp.diff(U, X) + sp.diff(V, Y)]
    f = [sp.lambdify((X, Y, Tt), e, "numpy") for e in ex]
    scn = S.mms_scenario()
    rng = np.random.default_rng(0)
    x, y = rng.uniform(0, 1, 64), rng.uniform(0, 1, 64)
    Fx, Fy = scn.forcing(x, y, 0.37)
    assert np.abs(Fx - f[0](x, y, 0.37)).max() < 1e-13
    assert np.abs(Fy - f[1](x, y, 0.37)).max() < 1e-13
    assert np.abs(scn.mass_source(x, y, 0.37) - f[2](x, y, 0.37)).max() < 1e-13


def test_travel_forcing_matches_oracle_sympy():
    from oracle import qfswe_oracle as O
    a, b = S.perturbed_square_scenario(), O.travel_wave()
    rng = np.random.default_rng(1)
    x, y = rng.uniform(0, 1000, 64), rng.uniform(0, 1000, 64)
    for p, q in zip(a.forcing(x, y, 12.5), b.forcing(x, y, 12.5)):
        assert np.abs(p - q).max() <= 1e-13 * np.abs(q).max()


def test_bump_fields_seeded_and_positive():
    xi0, hb, s = S.bump_fields(0)
    xi1, hb1, s1 = S.bump_fields(0)
    g = np.linspace(0, 1, 101)
    X, Y = np.meshgrid(g, g)
    assert s == s1 and np.array_equal(hb(X, Y), hb1(X, Y))
    assert hb(X, Y).min() >= 0.25 and 0 < xi0(X, Y).max() < 1


# ------------------------------------------------------- codegen / ABI
def test_codegen_deterministic_and_current():
    from paper_1904_08684_b200 import codegen
    for k in range(5):
        src = codegen.gen_order(k)
        assert src == codegen.gen_order(k)
        p = codegen.GEN_DIR / f"qf_order{k}.cuh"
        assert p.read_text() == src, "generated headers are stale: run codegen"


def test_cabi_exports_every_header_symbol():
    from paper_1904_08684_b200 import _cabi
    hdr = open(os.path.join(ROOT, "include", "qfswe.h")).read()
    names = set(re.findall(r"\b(qf_[a-z0-9_]+)\s*\(", hdr))
    assert names == set(_cabi.EXPORTS)
    lib = _cabi.load()
    for n in names:
        assert hasattr(lib, n), n
    assert lib.qf_abi_version() == 3


def test_locality_order_is_a_compact_permutation():
    m = M.build_unit_square_mesh(32)
    p = M.locality_order(m)
    assert np.array_equal(np.sort(p), np.arange(m.n_triangles))
    # blocks of 128 consecutive slots: most neighbours stay inside the block
    inv = np.empty_like(p)
    inv[p] = np.arange(len(p))
    nb = m.conn.nbr
    inside = 0
    total = 0
    for b0 in range(0, len(p), 128):
        el = p[b0:b0 + 128]
        n = nb[el]
        ok = n >= 0
        total += ok.sum()
        inside += ((inv[np.maximum(n, 0)] // 128 == b0 // 128) & ok).sum()
    assert inside / total > 0.8
