"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (needs /root/reference, read-only):

    python tests/golden/make_golden.py                 # all fixtures
    python tests/golden/make_golden.py --mass-flux     # massflux_k*.npz only

It imports the reference package under the alias ``qfswe_ref`` (it has no
``__init__.py``) and writes small ``.npz`` fixtures next to this
script.  The BASELINE manufactured solution is not admissible in the
reference as shipped (scenario.py:72-77 rejects a non-zero mass residual),
so the C1 case runs through the documented oracle extension: a subclass of
the reference ``Discretization`` whose ``source_rhs`` adds the projected xi
mass source, and a scenario built with ``manufacture=False`` whose momentum
forcing follows the reference formula (scenario.py:78-93).
"""

from __future__ import annotations

import importlib
import sys
import types
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = "/root/reference/pkg/src/qfswe"


def load_reference():
    if "qfswe_ref" not in sys.modules:
        pkg = types.ModuleType("qfswe_ref")
        pkg.__path__ = [REF]
        sys.modules["qfswe_ref"] = pkg
    return types.SimpleNamespace(**{
        n: importlib.import_module(f"qfswe_ref.{n}")
        for n in ("symbolic", "tensors", "mesh", "scenario", "solver", "harness")})


def unit_square(R, n):
    """BASELINE SW-NE split unit-square mesh, built as reference Mesh objects."""
    xs = np.linspace(0.0, 1.0, n + 1)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    verts = np.column_stack([X.ravel(), Y.ravel()])
    tris = []
    for i in range(n):
        for j in range(n):
            v00, v10 = i * (n + 1) + j, (i + 1) * (n + 1) + j
            v11, v01 = (i + 1) * (n + 1) + j + 1, i * (n + 1) + j + 1
            tris += [(v00, v10, v11), (v00, v11, v01)]
    mesh = R.mesh.Mesh(vertices=verts, triangles=np.array(tris, dtype=np.int64))
    R.mesh._build_edges(mesh)
    return mesh


def mms_scenario(R, **kw):
    """BASELINE MMS as a reference Scenario (forcing per scenario.py:78-93)."""
    import sympy as sp

    S = R.scenario
    X, Y, T = S.X, S.Y, S.T
    xi = sp.sin(2 * sp.pi * (X + Y - T)) / 100
    hb = 1 + X * Y / 10
    H = hb + xi
    U = H * sp.cos(2 * sp.pi * (X - T)) / 10
    V = H * sp.sin(2 * sp.pi * (Y - T)) / 10
    scn = S._build("mms", xi, U, V, hb, manufacture=False, **kw)
    g = sp.Float(scn.g)
    Fx = sp.diff(U, T) + sp.diff(U**2 / H, X) + sp.diff(U * V / H, Y) + g * H * sp.diff(xi, X)
    Fy = sp.diff(V, T) + sp.diff(U * V / H, X) + sp.diff(V**2 / H, Y) + g * H * sp.diff(xi, Y)
    scn.forcing = S._lambdify((X, Y, T), [Fx, Fy])
    mass = S._lambdify((X, Y, T), [sp.diff(xi, T) + sp.diff(U, X) + sp.diff(V, Y)])
    scn.mass_source = lambda x, y, t: mass(x, y, t)[0]
    return scn


def mms_discretization(R):
    class MassSourceDiscretization(R.solver.Discretization):
        """Oracle extension: xi mass source projected like solver.py:719-724."""

        def source_rhs(self, state, t):
            out = super().source_rhs(state, t)
            x, y = self.quad_xy[:, :, 0], self.quad_xy[:, :, 1]
            S = self.scn.mass_source(x, y, t)
            out[:, 0] += self.geom.sqrt_detB[:, None] * ((S * self.quad_w) @ self.quad_phi.T)
            return out
    return MassSourceDiscretization


def wall_discretization(R):
    """Oracle extension for the BASELINE C3-C5 physics: every boundary edge
    is a reflective wall.

    * The wall marker is admitted past the Dirichlet-only check of
      ``_setup_edges`` (solver.py:174-179) by handing the reference a
      scenario whose ``dirichlet_markers`` contain it; the boundary pass
      (``pass_B``) is then built as usual and only its use changes.
    * ``_boundary_flux`` (solver.py:622-688): the ghost state is the mirror
      image of the own state, xi+ = xi-, q+ = q- - 2 (q-.n) n, u+ likewise.
      The normal is constant along a straight edge, so the mirrored
      coefficient vectors have exactly the mirrored traces; the LF flux is
      then assembled with the reference's own pair/triple primitives and
      scalings, the ghost using the element's own h_b (as the Dirichlet
      ghost does, solver.py:668).
    * ``compute_lambda`` boundary branch (solver.py:374-405): the mirror has
      the same depth and |u.n|, so the wall edge's speed is the own side's
      maximum; DryState when the own depth is non-positive.
    """
    import dataclasses

    XI, U, V = 0, 1, 2

    class WallDiscretization(R.solver.Discretization):
        def compute_lambda(self, state, t):
            pb = self.pass_B
            self.pass_B = dataclasses.replace(pb, edge_index=pb.edge_index[:0])
            try:
                lam = super().compute_lambda(state, t)
            finally:
                self.pass_B = pb
            g, sd = self.scn.g, self.geom.sqrt_detB
            for e_t, rows in pb.groups.items():
                el = pb.elem[rows]
                tr = self.trace_at_samples[e_t]
                s = sd[el][:, None]
                H = ((self.hb_coef[el] + state.c[el, XI]) @ tr) / s
                un = ((state.u[el, 0] @ tr) * pb.n1[rows, None]
                      + (state.u[el, 1] @ tr) * pb.n2[rows, None]) / s
                if (H <= 0.0).any():
                    raise R.solver.DryState("non-positive depth at a wall edge sample")
                lam[pb.edge_index[rows]] = (np.abs(un) + np.sqrt(g * H)).max(axis=1)
            return lam

        def _boundary_flux(self, state, t, lam, rhs):
            assert self.scn.hb_mode == "linear"
            pb = self.pass_B
            g, sd, det = self.scn.g, self.geom.sqrt_detB, self.geom.detB
            c, u, hb = state.c, state.u, self.hb_coef
            for e_t, rows in pb.groups.items():
                ec = pb.elem[rows]
                n1, n2 = pb.n1[rows][:, None], pb.n2[rows][:, None]
                ln = pb.length[rows][:, None]
                lm = lam[pb.edge_index[rows]][:, None]

                def mirror(a, b):
                    dn = n1 * a + n2 * b
                    return a - 2.0 * n1 * dn, b - 2.0 * n2 * dn

                own = (c[ec, XI], c[ec, U], c[ec, V], u[ec, 0], u[ec, 1])
                ghost = (c[ec, XI], *mirror(c[ec, U], c[ec, V]), *mirror(u[ec, 0], u[ec, 1]))
                ip = (1.0 / det[ec])[:, None]
                it = (1.0 / (det[ec] * sd[ec]))[:, None]
                lin, quad = [], []
                for xi, qx, qy, vx, vy in (own, ghost):
                    lin.append([self._pair_own(e_t, f) * ip for f in (xi, qx, qy)])
                    pres = [(xi, xi, 0.5 * g), (xi, hb[ec], g)]
                    quad.append([
                        self._triple_own(e_t, [(qx, vx, 1.0)] + pres) * it,
                        self._triple_own(e_t, [(qx, vy, 1.0)]) * it,
                        self._triple_own(e_t, [(qy, vx, 1.0)]) * it,
                        self._triple_own(e_t, [(qy, vy, 1.0)] + pres) * it,
                    ])
                (xo, Uo, Vo), (xg, Ug, Vg) = lin
                A, B_, C_, D = (quad[0][i] + quad[1][i] for i in range(4))
                f_xi = 0.5 * (n1 * (Uo + Ug) + n2 * (Vo + Vg)) + 0.5 * lm * (xo - xg)
                f_U = 0.5 * (n1 * A + n2 * B_) + 0.5 * lm * (Uo - Ug)
                f_V = 0.5 * (n1 * C_ + n2 * D) + 0.5 * lm * (Vo - Vg)
                rhs[ec] -= np.stack([f_xi, f_U, f_V], axis=1) * ln[:, :, None]

    return WallDiscretization


def wall_runs(R):
    """BASELINE C3/C4 physics (bumps at rest, seeded sine bathymetry,
    reflective walls, CFL time step) and the C2 schedule, run by the
    reference at reduced N but at the stated step counts:

    * walls_p3_n16.npz : C3 shape, p = 3, uniform N = 16, 500 steps
    * walls_p2_j16.npz : C4 shape, p = 2, N = 16 jittered 0.2 h (seed 7), 300 steps
    * mms_p2_n16.npz   : C2 shape, p = 2, N = 16, SSP-RK3, dt = 2e-5, 1000 steps

    The bump / bathymetry callables and the mesh vertices come from this
    repository's generators (the reference has none for them); the fixture
    stores the vertices so the test can check the generator reproduces them.
    dt = 0.1 h_min / ((2k + 1) lambda_max(t = 0)) with the reference's h_min
    (solver.py:240-246) and wall lambda; the GPU test checks its own dt
    against the stored one.
    """
    import time

    sys.path.insert(0, str(HERE.parent.parent))
    from paper_1904_08684_b200 import mesh as M, scenario as S

    Wall = wall_discretization(R)
    xi0, hb, used = S.bump_fields(0)
    cases = (("walls_p3_n16", 3, M.build_unit_square_mesh(16), 500),
             ("walls_p2_j16", 2, M.build_unit_square_mesh(16, jitter=0.2, seed=7), 300))
    for name, k, m, steps in cases:
        t0 = time.time()
        mesh = R.mesh.Mesh(vertices=m.vertices.copy(), triangles=m.triangles.copy())
        R.mesh._build_edges(mesh)
        scn = R.scenario.Scenario(name="bumps", dt=1.0, dirichlet_markers=frozenset({1}), hb=hb)
        disc = Wall(mesh, scn, k)
        c0 = np.zeros((mesh.n_triangles, 3, disc.K))
        c0[:, 0] = disc.project_volume(xi0)
        st0 = R.solver.State(c=c0, u=np.zeros((mesh.n_triangles, 2, disc.K)), t=0.0)
        disc.solve_velocity(st0)
        lam0 = disc.compute_lambda(st0, 0.0)
        dt = 0.1 * disc.h_min / ((2 * k + 1) * float(lam0.max()))
        scn.dt = dt
        terms = stage_terms(disc, st0, 0.0)
        st = st0
        snaps = {}
        for i in range(1, steps + 1):
            st = disc.step(st)
            if i in (1, 10):
                snaps[f"c{i}"] = st.c
        np.savez_compressed(HERE / f"{name}.npz", verts=m.vertices, c0=st0.c, u0=st0.u,
                            cN=st.c, uN=st.u, steps=steps, dt=dt, h_min=disc.h_min, seed=used,
                            rhs0=disc.rhs(st0, 0.0), **snaps, **terms)
        print(f"{name}: {steps} steps, dt={dt:.6e}, {time.time() - t0:.1f} s")
    # C2 schedule at N = 16
    t0 = time.time()
    Disc = mms_discretization(R)
    disc = Disc(unit_square(R, 16), mms_scenario(R, dt=2e-5, t_end=1000 * 2e-5), 2)
    st0 = disc.project_initial()
    st = disc.run(st0)
    err = R.harness.l2_error(disc, st, st.t)
    np.savez_compressed(HERE / "mms_p2_n16.npz", c0=st0.c, cN=st.c, uN=st.u, t=st.t, steps=1000,
                        err=np.array(err.errors()))
    print(f"mms_p2_n16: 1000 steps, {time.time() - t0:.1f} s")


def format_files(R):
    """Files written by the reference's own writers (byte-comparison fixtures,
    tests/golden/formats/): ``save_mesh`` (mesh.py:285-301) of the perturbed
    square level 2 and of a jittered unit-square mesh, ``write_vtk``
    (harness.py:151-189) of the square_k2 perturbed state, and
    ``ConvergenceTable.to_csv`` (harness.py:57-68) of the sweep_p1 errors."""
    sys.path.insert(0, str(HERE.parent.parent))
    from paper_1904_08684_b200 import mesh as M

    out = HERE / "formats"
    out.mkdir(exist_ok=True)
    R.mesh.save_mesh(R.mesh.build_square_mesh(2, 0.2, 5), out / "square_l2.mesh")
    m = M.build_unit_square_mesh(4, jitter=0.2, seed=7)
    rm = R.mesh.Mesh(vertices=m.vertices.copy(), triangles=m.triangles.copy())
    R.mesh._build_edges(rm)
    R.mesh.save_mesh(rm, out / "unit4_jitter.mesh")
    g = np.load(HERE / "square_k2.npz")
    disc = R.solver.Discretization(R.mesh.build_square_mesh(3, 0.2, 42),
                                   R.scenario.perturbed_square_scenario(dt=0.5), 2)
    R.harness.write_vtk(disc, R.solver.State(c=g["cr"], u=g["ur"], t=0.0), out / "square_k2.vtk")
    sw = np.load(HERE / "sweep_p1.npz")
    rows = [R.harness.ErrorReport(order=1, level=int(n), elements=2 * int(n) ** 2,
                                  err_xi=float(e[0]), err_U=float(e[1]), err_V=float(e[2]))
            for n, e in zip(sw["n"], sw["err"])]
    (out / "sweep_p1.csv").write_text(R.harness.ConvergenceTable(rows=rows).to_csv())


CUSTOM_FIELDS = ("sin(x/300 - t/10)/100", "0.3*sin(x/300 - t/10) + 0.1", "0.05*cos(x/500)",
                 "2 + x/2000 + y/3000")


def custom_runs(R):
    """Reference ``custom_scenario`` (scenario.py:153-157; Dirichlet data from
    the fields, momentum forcing manufactured by SymPy) on the perturbed
    square, k = 1..3: terms on a perturbed state and 5 steps."""
    mesh = R.mesh.build_square_mesh(3, 0.2, 42)
    for k in (1, 2, 3):
        scn = R.scenario.custom_scenario(*CUSTOM_FIELDS, dt=0.5)
        disc = R.solver.Discretization(mesh, scn, k)
        st0 = disc.project_initial()
        sr = perturbed_state(disc, st0, 500 + k)
        terms = stage_terms(disc, sr, 2.3)
        st = st0
        for _ in range(5):
            st = disc.step(st)
        np.savez_compressed(HERE / f"custom_k{k}.npz", c0=st0.c, cr=sr.c, ur=sr.u,
                            rhs_r=disc.rhs(sr, 2.3), c5=st.c, u5=st.u, **terms)


def stage_terms(disc, state, t):
    lam = disc.compute_lambda(state, t)
    return dict(lam=lam, elem=disc.element_rhs(state), edge=disc.edge_rhs(state, t, lam),
                src=disc.source_rhs(state, t))


def perturbed_state(disc, state, seed):
    rng = np.random.default_rng(seed)
    c = state.c * (1.0 + 0.05 * rng.standard_normal(state.c.shape))
    s = type(state)(c=c, u=np.zeros_like(state.u), t=state.t)
    disc.solve_velocity(s)
    return s


def tensor_files(R):
    """verify_tensors reports and SHA-256 of every dump_tensors_csv file, k = 0..3."""
    import hashlib
    import tempfile

    out = {}
    for k in range(4):
        t = R.tensors.build_ref_tensors(k)
        if k > 0:  # the reference's verify_tensors divides by max|S| = 0 at k = 0
            rep = R.tensors.verify_tensors(t)
            out[f"report_k{k}"] = np.array([rep.max_abs_dev, rep.max_rel_dev])
        with tempfile.TemporaryDirectory() as d:
            for path in R.tensors.dump_tensors_csv(t, d):
                out[f"sha_{path.stem}"] = np.array(hashlib.sha256(path.read_bytes()).hexdigest())
    np.savez_compressed(HERE / "tensor_files.npz", **out)


def mass_flux(R):
    """instrument_mass_flux / last_mass_flux of edge_rhs (solver.py:123-124,
    619-620, 696-701) on the perturbed states of square_k{k}.npz, k = 1..3."""
    mesh = R.mesh.build_square_mesh(3, 0.2, 42)
    for k in (1, 2, 3):
        g = np.load(HERE / f"square_k{k}.npz")
        disc = R.solver.Discretization(mesh, R.scenario.perturbed_square_scenario(dt=0.5), k)
        disc.instrument_mass_flux = True
        st = R.solver.State(c=g["cr"].copy(), u=g["ur"].copy(), t=0.0)
        disc.edge_rhs(st, 3.7)
        mL, mR = disc.last_mass_flux
        np.savez_compressed(HERE / f"massflux_k{k}.npz", mL=mL, mR=mR)


def main():
    R = load_reference()
    if "--tensor-files" in sys.argv:
        return tensor_files(R)
    if "--mass-flux" in sys.argv:
        return mass_flux(R)
    if "--walls" in sys.argv:
        return wall_runs(R)
    if "--formats" in sys.argv:
        return format_files(R)
    if "--custom" in sys.argv:
        return custom_runs(R)
    # A. tensors
    for k in range(4):
        t = R.tensors.build_ref_tensors(k)
        np.savez_compressed(HERE / f"tensors_k{k}.npz", **t.as_dict())
    # B. reference-native perturbed square, k = 0..3
    mesh = R.mesh.build_square_mesh(3, 0.2, 42)
    for k in range(4):
        scn = R.scenario.perturbed_square_scenario(dt=0.5)
        disc = R.solver.Discretization(mesh, scn, k)
        st0 = disc.project_initial()
        sr = perturbed_state(disc, st0, 100 + k)
        terms = stage_terms(disc, sr, 3.7)
        st = st0
        for _ in range(3):
            st = disc.step(st)
        np.savez_compressed(HERE / f"square_k{k}.npz", c0=st0.c, u0=st0.u, cr=sr.c, ur=sr.u,
                            rhs_r=disc.rhs(sr, 3.7), c3=st.c, u3=st.u, **terms)
    # C. lake at rest
    mesh2 = R.mesh.build_square_mesh(2, 0.2, 5)
    for k in (1, 2, 3):
        scn = R.scenario.lake_at_rest_scenario(dt=0.5)
        disc = R.solver.Discretization(mesh2, scn, k)
        st0 = disc.project_initial()
        st = st0
        for _ in range(10):
            st = disc.step(st)
        np.savez_compressed(HERE / f"lake_k{k}.npz", c0=st0.c, rhs0=disc.rhs(st0, 0.0), c10=st.c)
    # D. BASELINE C1 in full (MMS + mass source, p=1, N=32, RK2, 200 steps)
    Disc = mms_discretization(R)
    m32 = unit_square(R, 32)
    scn = mms_scenario(R, dt=1e-4, t_end=0.02)
    disc = Disc(m32, scn, 1)
    st0 = disc.project_initial()
    terms = stage_terms(disc, st0, 0.0)
    st = disc.run(st0)
    err = R.harness.l2_error(disc, st, st.t)
    np.savez_compressed(HERE / "c1_mms_p1_n32.npz", c0=st0.c, u0=st0.u, c200=st.c, u200=st.u,
                        t=st.t, err=np.array(err.errors()), **terms)
    # E. small MMS p = 2, 3 (C2 shape at reduced size)
    for k, n, steps in ((2, 8, 20), (3, 6, 10)):
        m = unit_square(R, n)
        scn = mms_scenario(R, dt=2e-5)
        disc = Disc(m, scn, k)
        st0 = disc.project_initial()
        sr = perturbed_state(disc, st0, 7 + k)
        terms = stage_terms(disc, sr, 0.3)
        st = st0
        for _ in range(steps):
            st = disc.step(st)
        np.savez_compressed(HERE / f"mms_p{k}_n{n}.npz", c0=st0.c, cr=sr.c, ur=sr.u,
                            cN=st.c, uN=st.u, steps=steps, **terms)
    # F. ring level 2, k = 1
    mr = R.mesh.build_ring_mesh(2)
    scn = R.scenario.ring_scenario(dt=0.5)
    disc = R.solver.Discretization(mr, scn, 1)
    st0 = disc.project_initial()
    terms = stage_terms(disc, st0, 0.0)
    st = disc.step(disc.step(st0))
    np.savez_compressed(HERE / "ring_k1.npz", c0=st0.c, c2=st.c, **terms)
    # H. hb_mode = "const" (paper-form bathymetry, solver.py:498-510, 606-608)
    for k in (1, 2):
        scn = R.scenario.perturbed_square_scenario(dt=0.5, hb_mode="const")
        disc = R.solver.Discretization(mesh, scn, k)
        st0 = disc.project_initial()
        sr = perturbed_state(disc, st0, 300 + k)
        terms = stage_terms(disc, sr, 1.3)
        st = disc.step(disc.step(st0))
        np.savez_compressed(HERE / f"const_k{k}.npz", cr=sr.c, ur=sr.u, c2=st.c, **terms)
    # G. MMS convergence sweeps (reference errors for the EOC tests)
    for k, ns, dt, steps in ((1, (8, 16, 32), 1e-4, 200), (2, (8, 16), 2e-5, 200),
                             (3, (4, 8), 2e-5, 100)):
        errs = []
        for n in ns:
            m = unit_square(R, n)
            scn = mms_scenario(R, dt=dt, t_end=steps * dt)
            disc = Disc(m, scn, k)
            st = disc.run()
            errs.append(R.harness.l2_error(disc, st, st.t).errors())
        np.savez_compressed(HERE / f"sweep_p{k}.npz", n=np.array(ns), err=np.array(errs),
                            dt=dt, steps=steps)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
