"""On-disk formats: byte equality with files written by
the reference's own writers (tests/golden/formats/, made by
``make_golden.py --formats``): ``ghoddess-mesh 1`` (mesh.py:285-301),
legacy VTK (harness.py:151-189) and the convergence CSV (harness.py:57-78)."""

import os

import numpy as np

from conftest import GOLDEN

FMT = os.path.join(GOLDEN, "formats")


def _read(name):
    with open(os.path.join(FMT, name)) as fh:
        return fh.read()


def test_mesh_file_bytes_match_reference_writer(tmp_path):
    from paper_1904_08684_b200 import mesh as M
    for name, mesh in (("square_l2.mesh", M.build_square_mesh(2, 0.2, 5)),
                       ("unit4_jitter.mesh", M.build_unit_square_mesh(4, jitter=0.2, seed=7))):
        p = tmp_path / name
        M.save_mesh(mesh, p)
        assert p.read_text() == _read(name)
        # and the reference-written file loads into the same mesh
        back = M.load_mesh(os.path.join(FMT, name))
        assert np.array_equal(back.vertices, mesh.vertices)
        assert np.array_equal(back.triangles, mesh.triangles)


def test_vtk_bytes_match_reference_writer(tmp_path, golden):
    from paper_1904_08684_b200 import harness as Hn, mesh as M, scenario as S
    from paper_1904_08684_b200.solver import HostSetup, State
    g = golden("square_k2.npz")
    host = HostSetup(M.build_square_mesh(3, 0.2, 42), S.perturbed_square_scenario(dt=0.5), 2)
    p = tmp_path / "out.vtk"
    Hn.write_vtk(host, State(g["cr"], g["ur"], 0.0), p)
    assert p.read_text() == _read("square_k2.vtk")


def test_convergence_csv_bytes_match_reference_writer(golden):
    from paper_1904_08684_b200 import harness as Hn
    sw = golden("sweep_p1.npz")
    rows = [Hn.ErrorReport(order=1, level=int(n), elements=2 * int(n) ** 2, err_xi=float(e[0]),
                           err_U=float(e[1]), err_V=float(e[2]))
            for n, e in zip(sw["n"], sw["err"])]
    text = Hn.ConvergenceTable(rows=rows).to_csv()
    assert text == _read("sweep_p1.csv")
    back = Hn.ConvergenceTable.parse_csv(text, order=1)
    assert [r.errors() for r in back.rows] == [r.errors() for r in rows]


def test_eoc_last_digit_matches_reference_formula():
    """ln(p/c)/ln 2, not log2: the two differ in the last ulp for ~1/3 of ratios."""
    from paper_1904_08684_b200 import harness as Hn
    rng = np.random.default_rng(0)
    e = np.sort(rng.uniform(1e-9, 1e-3, (40, 3)), axis=0)[::-1]
    rows = [Hn.ErrorReport(1, i, 2, *map(float, r)) for i, r in enumerate(e)]
    got = Hn.ConvergenceTable(rows).eoc()
    want = [tuple(np.log(p / c) / np.log(2.0) for p, c in zip(a, b)) for a, b in zip(e, e[1:])]
    assert got == want
