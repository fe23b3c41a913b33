"""GPU parity at the BASELINE sizes against fixtures produced by the
reference itself (tests/golden/make_golden_large.py -> oracle/_ref):

* tree + interaction lists bit-exact (SHA-256 digest of perm, offsets, lists),
  C2-C5 (C5: the reference's build_tree + build_interaction_lists only);
* matvec within relative 2-norm 10 x eps of the reference's full matvec
  output (C2, C3, C4), and on the 2000 rows drawn by the reference's own
  sampling rule;
* error against the exact dense product no worse than 2 x the reference's,
  on those rows and through the device reference_error (the same estimator,
  hmatrix.cpp:253-291).
"""
import hashlib

import numpy as np
import pytest

from conftest import LARGE_NAMES, load_golden

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def digest(rep):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rep.perm(), dtype=np.int32).tobytes())
    for l in range(rep.depth + 1):
        h.update(np.ascontiguousarray(rep.offsets(l), dtype=np.int64).tobytes())
        if l >= 1:
            for k in range(3):
                o, ids = rep.list(l, k)
                h.update(np.ascontiguousarray(o, dtype=np.int32).tobytes())
                h.update(np.ascontiguousarray(ids, dtype=np.int32).tobytes())
    return h.hexdigest()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("policy", ["auto", "stream"])
@pytest.mark.parametrize("name", LARGE_NAMES)
def test_large_config_against_reference(h3d, name, policy):
    g = load_golden(f"large_{name}")
    if "tree_only" in g:
        pytest.skip("tree/list digest only (test_c5_on_one_gpu)")
    n, seed, eps = int(g["n"]), int(g["seed"]), float(g["eps"])
    pts = h3d.generate_points(n, seed)
    x = h3d.random_vector(n, seed + 17)
    rep = h3d.initialize(pts, h3d.make_kernel(str(g["kernel"])), "hodlr3d",
                         h3d.HmatOptions(n_max=int(g["n_max"]), epsilon=eps, mode_policy=policy))
    assert rep.depth == int(g["depth"])
    assert digest(rep) == str(g["tree_digest"]), "tree/lists must be bit-exact"
    b = rep.matvec(x)
    rows = g["rows"]
    if "b_ref" in g:
        assert rel(b, g["b_ref"]) <= 10 * eps
    assert rel(b[rows], g["b_ref_rows"]) <= 10 * eps
    err = rel(b[rows], g["b_exact_rows"])
    ref_err = rel(g["b_ref_rows"], g["b_exact_rows"])
    # the sampled-row error matches the reference's own reference_error (which sums
    # 1/sqrt(r^2) rows instead of eval_pair's 1/r: equal to ~1e-5 relative)
    assert abs(ref_err - float(g["ref_error"])) <= 1e-2 * float(g["ref_error"]) + 1e-14
    assert err <= 2 * ref_err, (err, ref_err)
    # the reference's estimator on the device (same 2000 rows, exact sums)
    dev_err = rep.reference_error(x, b)
    assert dev_err <= 2 * float(g["ref_error"]), (dev_err, float(g["ref_error"]))
    if policy == "stream":
        # ACA ranks per level against the reference's census (count, sum and
        # max of its ordered-block ranks). The reference compresses (X, Y) and
        # (Y, X) separately (each ACA starts from its own row 0, so the two
        # orientations' ranks can differ by a few); the device compresses each
        # unordered pair once, so 2 x its rank sum tracks the census sum.
        rows_out = []
        for l, cnt, rsum, rmax in g["ranks"]:
            _, _, r = rep.pairs(int(l))
            rows_out.append((int(l), int(cnt), int(rsum), int(rmax), len(r), 2 * int(r.sum()), int(r.max())))
            print(f"{name} level {l}: ref blocks {cnt} sum {rsum} max {rmax}; "
                  f"device pairs {len(r)} 2*sum {2 * int(r.sum())} max {int(r.max())}")
        for l, cnt, rsum, rmax, npair, dsum, dmax in rows_out:
            assert 2 * npair == cnt
            assert abs(dsum - rsum) <= (0.05 if cnt < 100 else 0.01) * rsum, l
            assert abs(dmax - rmax) <= max(2, 0.05 * rmax), l
    rep.close()


def test_c5_on_one_gpu(h3d, oracle):
    # BASELINE configs[4] (N = 4,194,304, Laplace, tol 1e-6, matrix-free near
    # field), the reference's 8-GPU case, fits one B200 in the hybrid
    # representation. The reference's full initialize needs ~66 GB and ~12
    # CPU-minutes of ACA, so the fixture holds its tree/list digest only
    # (bit-exact here); the matvec is checked by the reference's acceptance
    # form: reference_error (2000 rows of mt19937_64(7), exact sums,
    # hmatrix.cpp:253-291) within 10 x tol, cross-checked on 100 of those
    # rows by the CPU checker.
    g = load_golden("large_c5")
    n, eps = int(g["n"]), float(g["eps"])
    pts = h3d.generate_points(n, int(g["seed"]))
    x = h3d.random_vector(n, int(g["seed"]) + 17)
    rep = h3d.initialize(pts, h3d.make_kernel("laplace3d"), "hodlr3d",
                         h3d.HmatOptions(n_max=int(g["n_max"]), epsilon=eps, dense_mode="on-the-fly"))
    assert rep.depth == int(g["depth"]) == 6
    assert digest(rep) == str(g["tree_digest"]), "tree/lists must be bit-exact"
    b = rep.matvec(x)
    err = rep.reference_error(x, b)
    print(f"C5 reference_error {err:.3e} (tol {eps:g}), modes {rep.stats()['level_modes'][:7]}")
    assert err <= 10 * eps
    u = (h3d.random_vector(100, 7) + 1.0) / 2.0  # the first 100 of the reference's draws
    rows = rep.perm()[(u * n).astype(np.int64)]
    import os
    oracle.set_threads(os.cpu_count() or 1)
    ex = oracle.exact_rows(pts, x, rows)
    assert rel(b[rows], ex) <= 10 * eps
    rep.close()
