"""Device GMRES / integral-equation solver (SURVEY.md section 8(f) "next"):
reference solver.hpp / solver.cpp.

CPU tests pin the host helpers (cell self-integral, tensor grid) bit-exact to
the reference; GPU tests run the manufactured-solution experiment
(solver.cpp:243-300) through the C-ABI and compare it with the reference's own
results in tests/golden/ie_cases.json (tests/golden/make_ie_golden.py):
converged flag equal, iteration count within +-2, forward error no worse than
2x the reference's (floor 1e-13 for the near-exact cases).
"""
import json
from pathlib import Path

import numpy as np
import pytest

IE = json.loads((Path(__file__).resolve().parent / "golden" / "ie_cases.json").read_text())


def _pkg():
    import paper_2307_16303_b200 as pkg  # the library loads without a GPU
    return pkg


def test_cell_self_integral_matches_reference_golden():
    h3d = _pkg()
    for h, v in IE["cell_self_integral"]:
        assert h3d.cell_self_integral(h) == v, h


def test_unit_cell_constant_frozen():
    # test_solver.cpp:94-102
    h3d = _pkg()
    assert abs(h3d.cell_self_integral(1.0) - 2.380077363979) <= 2.380077363979 * 1e-9
    assert h3d.cell_self_integral(0.5) == pytest.approx(h3d.cell_self_integral(1.0) / 4, rel=1e-15)
    assert h3d.cell_self_integral(0.125) == pytest.approx(h3d.cell_self_integral(0.25) / 4, rel=1e-15)


def test_unit_cell_constant_against_closed_form():
    # integral of 1/|u| over [-1/2, 1/2]^3 = 3 ln(2 + sqrt 3) - pi/2 (the
    # reference's quadrature value is within a few ulp of it)
    import math
    h3d = _pkg()
    exact = 3 * math.log(2 + math.sqrt(3)) - math.pi / 2
    assert h3d.cell_self_integral(1.0) == pytest.approx(exact, rel=1e-14)


def test_cell_self_integral_scales_as_h_squared():
    h3d = _pkg()
    c = h3d.cell_self_integral(1.0)
    for h in (0.5, 0.125, 3.0):
        assert abs(h3d.cell_self_integral(h) - h * h * c) <= 1e-15 * h * h * c


def test_cell_self_integral_against_live_reference(ref):
    h3d = _pkg()
    for h in np.geomspace(1e-3, 4.0, 9):
        assert h3d.cell_self_integral(h) == ref.cell_self_integral(h)


@pytest.mark.parametrize("side", [1, 2, 5, 16])
def test_tensor_grid_matches_reference_order(side):
    h3d = _pkg()
    n = side ** 3
    p = h3d.generate_grid_points(n)
    c = -1.0 + (2.0 * np.arange(side) + 1.0) / side
    ix, iy, iz = np.meshgrid(c, c, c, indexing="ij")  # z fastest (kernel.cpp:104-107)
    want = np.stack([ix.ravel(), iy.ravel(), iz.ravel()], axis=1)
    assert np.array_equal(p, want)


def test_tensor_grid_live_reference(ref):
    h3d = _pkg()
    assert np.array_equal(h3d.generate_grid_points(343), ref.generate_points(343, 0, dist=1))


def test_tensor_grid_rejects_non_cube():
    h3d = _pkg()
    with pytest.raises(ValueError):
        h3d.generate_grid_points(100)


def test_discretize_ie_guards():
    h3d = _pkg()
    with pytest.raises(ValueError):
        h3d.discretize_ie(1, h3d.make_kernel("laplace3d"), 1e-7)
    with pytest.raises(ValueError):
        h3d.discretize_ie(8, h3d.make_kernel("r4"), 1e-7)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("case", IE["ie"], ids=lambda c: "n{grid_n}_eps{eps:g}_r{restart}_m{max_iter}".format(**c))
def test_ie_experiment_vs_reference(h3d, case):
    r = h3d.ie_experiment(case["grid_n"], h3d.make_kernel("laplace3d"), case["eps"], seed=case["seed"],
                          base=h3d.HmatOptions(n_max=case["n_max"]),
                          gmres_opt=h3d.GmresOptions(tol=case["tol"], restart=case["restart"],
                                                     max_iter=case["max_iter"]))
    assert r.size == case["grid_n"] ** 3
    if case["converged"]:
        assert r.converged
        assert abs(r.iterations - case["iterations"]) <= 2, (r.iterations, case["iterations"])
    elif case["max_iter"] < 50:
        # budget exhausted in both: same count, same (large) error scale
        assert not r.converged and r.iterations == case["max_iter"]
    assert r.forward_error <= max(2 * case["forward_error"], 1e-13), (r.forward_error, case)


@pytest.mark.gpu
def test_gmres_shifted_operator_vs_dense_solve(h3d, oracle):
    """(alpha I + beta A~) x = f against numpy's dense solve of the exact
    operator: agreement to the compression tolerance, monotone residuals."""
    n, eps = 3000, 1e-10
    pts = h3d.generate_points(n, 41)
    rep = h3d.initialize(pts, h3d.make_kernel("laplace3d"), "hodlr3d", h3d.HmatOptions(n_max=64, epsilon=eps))
    alpha, beta = 2.0, 1.0 / n
    f = h3d.random_vector(n, 43)
    sol = rep.gmres(f, alpha, beta, h3d.GmresOptions(tol=1e-12, max_iter=200))
    assert sol.converged and sol.final_relres < 1e-12
    hist = sol.residual_history
    assert len(hist) == sol.iterations and np.all(np.diff(hist) <= 1e-15)
    d = pts[:, None, :] - pts[None, :, :]
    r = np.sqrt((d * d).sum(-1))
    np.fill_diagonal(r, np.inf)
    A = alpha * np.eye(n) + beta / r
    x = np.linalg.solve(A, f)
    assert np.linalg.norm(sol.x - x) / np.linalg.norm(x) < 1e-9
    # the returned residual is the true one of the returned iterate
    res = f - (alpha * sol.x + beta * rep.matvec(sol.x))
    assert abs(np.linalg.norm(res) / np.linalg.norm(f) - sol.final_relres) < 1e-14


@pytest.mark.gpu
def test_gmres_restart_and_edge_cases(h3d):
    n = 2000
    pts = h3d.generate_points(n, 5)
    rep = h3d.initialize(pts, h3d.make_kernel("laplace3d"), "hodlr3d", h3d.HmatOptions(n_max=64, epsilon=1e-9))
    f = h3d.random_vector(n, 6)
    full = rep.gmres(f, 2.0, 1.0 / n, h3d.GmresOptions(tol=1e-11))
    rs = rep.gmres(f, 2.0, 1.0 / n, h3d.GmresOptions(tol=1e-11, restart=3))
    assert full.converged and rs.converged and rs.iterations >= full.iterations
    assert np.linalg.norm(rs.x - full.x) / np.linalg.norm(full.x) < 1e-9
    # bitwise reproducible
    again = rep.gmres(f, 2.0, 1.0 / n, h3d.GmresOptions(tol=1e-11))
    assert np.array_equal(again.x, full.x) and again.iterations == full.iterations
    # zero rhs: converged at once with x = 0 (solver.cpp:31-35)
    z = rep.gmres(np.zeros(n), 2.0, 1.0 / n)
    assert z.converged and z.iterations == 0 and not np.any(z.x)
    # budget exhausted: best iterate, converged = False
    one = rep.gmres(f, 2.0, 1.0 / n, h3d.GmresOptions(tol=1e-14, max_iter=2))
    assert not one.converged and one.iterations == 2 and len(one.residual_history) == 2
    with pytest.raises(ValueError):
        rep.gmres(f, options=h3d.GmresOptions(tol=0.0))
    with pytest.raises(ValueError):
        rep.gmres(f[:-1])


@pytest.mark.gpu
@pytest.mark.parametrize("kern", ["laplace3d", "r4", "helmholtz-re"])
def test_direct_matvec_vs_oracle(h3d, oracle, kern):
    n = 3000
    pts = h3d.generate_points(n, 9)
    x = h3d.random_vector(n, 10)
    rep = h3d.initialize(pts, h3d.make_kernel(kern), "hodlr3d", h3d.HmatOptions(n_max=100))
    b = rep.direct_matvec(x)
    want = oracle.dense_matvec(pts, x, kern)
    assert np.linalg.norm(b - want) / np.linalg.norm(want) < 1e-14


@pytest.mark.gpu
def test_gmres_identity_and_diagonal_one_iteration(h3d):
    # test_solver.cpp:11-35: alpha I (beta = 0) is solved in one iteration
    pts = h3d.generate_points(500, 3)
    rep = h3d.initialize(pts, h3d.make_kernel("laplace3d"), options=h3d.HmatOptions(n_max=64))
    f = h3d.random_vector(500, 4)
    for alpha in (1.0, 2.5):
        r = rep.gmres(f, alpha, 0.0)
        assert r.converged and r.iterations == 1
        assert np.allclose(r.x, f / alpha, rtol=1e-14, atol=0)


@pytest.mark.gpu
def test_ie_n2_matches_dense_assembly(h3d):
    # test_solver.cpp:104-133
    op = h3d.discretize_ie(2, h3d.make_kernel("laplace3d"), 1e-7)
    try:
        assert op.size == 8
        assert op.diagonal == pytest.approx(1.0 + h3d.cell_self_integral(1.0))
        a = op.dense_matrix()
        p = op.collocation
        for i in range(8):
            for j in range(8):
                want = op.diagonal if i == j else op.cell_volume / np.linalg.norm(p[i] - p[j])
                assert a[i, j] == pytest.approx(want, rel=1e-14)
        x = np.random.default_rng(2).random(8)
        assert np.allclose(op.apply(x), a @ x, rtol=1e-6)
    finally:
        op.close()


@pytest.mark.gpu
def test_ie_hierarchical_apply_vs_dense(h3d):
    # test_solver.cpp:144-164
    eps = 1e-7
    op = h3d.discretize_ie(8, h3d.make_kernel("laplace3d"), eps)
    try:
        a = op.dense_matrix()
        rng = np.random.default_rng(12)
        for _ in range(3):
            x = 2 * rng.random(op.size) - 1
            y, ye = op.apply(x), a @ x
            assert np.linalg.norm(y - ye) / np.linalg.norm(ye) <= 10 * eps
    finally:
        op.close()


@pytest.mark.gpu
def test_ie_manufactured_solution_vs_dense_lu(h3d):
    # test_solver.cpp:166-190
    lap = h3d.make_kernel("laplace3d")
    rep = h3d.ie_experiment(8, lap, 1e-7, seed=99)
    assert rep.converged and rep.forward_error <= 1e-5
    op = h3d.discretize_ie(8, lap, 1e-7)
    try:
        sigma = h3d.random_vector(op.size, 99)
        a = op.dense_matrix()
        sc = np.linalg.solve(a, a @ sigma)
        dense_err = np.linalg.norm(sc - sigma) / np.linalg.norm(sigma)
        assert rep.forward_error <= max(10 * dense_err, 1e-5)
    finally:
        op.close()


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["hodlr", "hstrong"])
def test_ie_experiment_other_variants(h3d, variant):
    # the solver runs over every block structure (solver.cpp:218-240 takes a Variant)
    r = h3d.ie_experiment(12, h3d.make_kernel("laplace3d"), 1e-7, variant, seed=5,
                          base=h3d.HmatOptions(n_max=64))
    assert r.converged and r.forward_error <= 1e-7
