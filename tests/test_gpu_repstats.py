"""GPU: RepStats and reference_error against the reference.

* stats() follows RepStats (hmatrix.cpp:228-251): float_count = r^2 per
  ordered low-rank block + dense leaf areas, int_count = 2 r per block,
  memory = 8 floats + 4 ints, compression = floats / N^2.
* reference_error() follows hmatrix.cpp:253-291: exact row sums of every row
  for N <= 4096, else 2000 Morton rows drawn by mt19937_64(7).
"""
import numpy as np
import pytest

from conftest import GOLDEN_NAMES, load_golden

pytestmark = pytest.mark.gpu


def _rep(h3d, g, policy="stream", **kw):
    pts = h3d.generate_points(int(g["n"]), int(g["seed"]))
    opt = h3d.HmatOptions(n_max=int(g["n_max"]), epsilon=float(g["eps"]), mode_policy=policy,
                          max_rank=int(g.get("max_rank", 0)), **kw)
    return h3d.initialize(pts, h3d.make_kernel(str(g["kernel"]), float(g.get("diag", 0.0))),
                          str(g.get("variant", "hodlr3d")), opt)


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_repstats_against_reference(h3d, name):
    """Every level compressed (policy "stream"): the reference's dense-area
    part exactly; the rank part from the pairs this engine compressed (one ACA
    per unordered pair, applied in both orientations), which equals the
    reference's ordered-block sums exactly where the reference's two
    orientations got equal ranks and within 1 % overall."""
    g = load_golden(name)
    ref_float, ref_int, ref_mem, ref_maxr, ref_depth = (int(v) for v in g["stats"])
    rep = _rep(h3d, g)
    st = rep.stats()
    L = st["depth"]
    assert L == ref_depth
    ref_r2 = sum(int((g[f"lr_r{l}"].astype(np.int64) ** 2).sum()) for l in range(1, L + 1))
    ref_dense = ref_float - ref_r2
    pair_r2, pair_r = 0, 0
    for l in range(1, L + 1):
        _, _, r = rep.pairs(l)
        pair_r2 += int((r.astype(np.int64) ** 2).sum())
        pair_r += int(r.sum())
    assert st["ref_float_count"] == 2 * pair_r2 + ref_dense
    assert st["ref_int_count"] == 4 * pair_r
    assert st["max_rank"] <= ref_maxr + max(2, ref_maxr // 20)
    if ref_float:
        assert abs(st["ref_float_count"] - ref_float) <= 0.01 * ref_float
    if ref_int:
        assert abs(st["ref_int_count"] - ref_int) <= 0.01 * ref_int
    n = int(g["n"])
    assert st["compression_ratio"] == pytest.approx(st["ref_float_count"] / (n * n), rel=1e-12)
    # against the reference's own ordered ranks, pair by pair (X < Y)
    for l in range(1, L + 1):
        x, y, r = rep.pairs(l)
        ref = {(int(a), int(b)): int(c) for a, b, c in zip(g[f"lr_t{l}"], g[f"lr_s{l}"], g[f"lr_r{l}"])}
        if len(x) == 0:
            continue
        got = np.array([r[k] - ref[(int(x[k]), int(y[k]))] for k in range(len(x))])
        assert (np.abs(got) <= 2).all() and (got == 0).mean() >= 0.95, l


def test_storage_accounting(h3d):
    """test_hmatrix.cpp:155-176: float_count = sum r^2 + dense areas; the
    strong-admissibility structure within 2x; compression falls as N grows 8x."""
    lap = h3d.make_kernel("laplace3d")
    opt = h3d.HmatOptions(epsilon=1e-6, mode_policy="stream")
    pts = h3d.generate_points(8000, 41)
    s3 = h3d.initialize(pts, lap, "hodlr3d", opt).stats()
    assert s3["compression_ratio"] < 1.0
    ss = h3d.initialize(pts, lap, "hstrong", opt).stats()
    assert ss["ref_float_count"] < 2 * s3["ref_float_count"]
    assert s3["ref_float_count"] < 2 * ss["ref_float_count"]
    big = h3d.initialize(h3d.generate_points(64000, 41), lap, "hodlr3d", opt).stats()
    assert big["compression_ratio"] < s3["compression_ratio"]


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_reference_error_matches_reference(h3d, name):
    """Same rows as the reference (all rows up to N = 4096, else the 2000
    mt19937_64(7) draws), exact sums on the device: the reference's own
    reference_error(b_ref) value to summation-order rounding."""
    g = load_golden(name)
    rep = _rep(h3d, g, policy="auto")
    got = rep.reference_error(g["x"], g["b_ref"])
    # same rows; the exact row sums differ from the reference's sequential
    # sums by rounding (~1e-16 relative), which moves an error of size e by
    # ~1e-16 / e relative: 1e-6 separates "same rows" from any other draw
    assert got == pytest.approx(float(g["ref_error"]), rel=1e-6, abs=1e-13)


def test_reference_error_agrees_with_dense_at_small_n(h3d, oracle):
    """test_hmatrix.cpp:178-190."""
    pts = h3d.generate_points(1200, 43)
    rep = h3d.initialize(pts, h3d.make_kernel("laplace3d"), "hodlr3d",
                         h3d.HmatOptions(n_max=80, epsilon=1e-7))
    x = h3d.random_vector(1200, 6)
    b = rep.matvec(x)
    bex = oracle.dense_matvec(pts, x)
    err_orac = float(np.linalg.norm(b - bex) / np.linalg.norm(bex))
    assert rep.reference_error(x, b) == pytest.approx(err_orac, rel=1e-6)


def test_reference_error_sampled_rows_match_the_reference_rule(h3d, oracle):
    """N > exact_limit: the rows are floor(uniform01(mt19937_64(seed)) * N)
    Morton positions (hmatrix.cpp:264-271); recompute that estimator from
    exact row sums of the checker and compare."""
    n = 20000
    pts = h3d.generate_points(n, 5)
    rep = h3d.initialize(pts, h3d.make_kernel("r4"), "hodlr3d", h3d.HmatOptions(n_max=64, epsilon=1e-8))
    x = h3d.random_vector(n, 22)
    b = rep.matvec(x)
    for seed, rows in ((7, 2000), (123, 500)):
        u = (h3d.random_vector(rows, seed) + 1.0) / 2.0  # the same mt19937_64 draws, exactly
        pos = (u * n).astype(np.int64)
        orig = rep.perm()[pos]
        ex = oracle.exact_rows(pts, x, orig, "r4")
        want = float(np.sqrt(((b[orig] - ex) ** 2).sum() / (ex ** 2).sum()))
        got = rep.reference_error(x, b, sample_rows=rows, seed=seed)
        assert got == pytest.approx(want, rel=1e-6)
    # exact_limit above N: every row
    full = rep.reference_error(x, b, exact_limit=n)
    bex = oracle.dense_matvec(pts, x, "r4")
    assert full == pytest.approx(float(np.linalg.norm(b - bex) / np.linalg.norm(bex)), rel=1e-6)
