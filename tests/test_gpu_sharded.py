"""The sharded (multi-GPU) engine path on one GPU: every Morton-subtree shard
of a world of 2/4/8 is built in turn on cuda:0 (no communicator: x is
replicated, so the NCCL all-gather is the only piece not exercised here; the
plan and the exchange are covered on CPU by test_shard_plan.py with gloo).
Each shard's owned rows must reproduce the single-GPU matvec (the shards
compress the same pairs with the same deterministic kernels), mirroring the
reference's parallel-vs-serial check (test_parallel.cpp:89-102, <= 1e-12).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, SEED = 20000, 53


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("levels", [(0, 0, 0, 0), (0, 1, 0, 2), (0, 1, 1, 1), (0, 3, 3, 2), (0, 1, 3, 3),
                                    (0, 1, 4, 4), (0, 1, 4, 2), (0, 5, 1, 5), (0, 1, 5, 2), (0, 6, 6, 2), (0, 6, 1, 5)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_shards_reproduce_single_gpu(h3d, oracle, world, levels):
    pts = h3d.generate_points(N, SEED)
    x = h3d.random_vector(N, 9)
    opt = h3d.HmatOptions(n_max=64, epsilon=1e-7, mode_policy="explicit", level_modes=levels)
    lap = h3d.make_kernel("laplace3d")
    ref = h3d.initialize(pts, lap, options=opt)
    assert ref.depth == 3
    b1 = ref.matvec(x)
    perm = ref.perm()
    b = np.full(N, np.nan)
    rows_seen = 0
    for r in range(world):
        rep = h3d.initialize(pts, lap, options=opt, shard_rank=r, shard_world=world)
        st = rep.stats()
        own = perm[st["owned_row_begin"]:st["owned_row_end"]]
        rows_seen += len(own)
        b[own] = rep.matvec(x)[own]
        rep.close()
    assert rows_seen == N and not np.isnan(b).any()
    assert rel(b, b1) <= 1e-12
    assert rel(b, oracle.dense_matvec(pts, x)) <= 10 * opt.epsilon


@pytest.mark.parametrize("variant", ["hodlr", "hstrong"])
@pytest.mark.parametrize("world", [2, 8])
def test_shards_reproduce_single_gpu_variants(h3d, oracle, world, variant):
    # test_parallel.cpp:175-187 runs the parallel path on hstrong as well
    pts = h3d.generate_points(N, SEED)
    x = h3d.random_vector(N, 9)
    opt = h3d.HmatOptions(n_max=64, epsilon=1e-7)
    lap = h3d.make_kernel("laplace3d")
    ref = h3d.initialize(pts, lap, variant, options=opt)
    b1 = ref.matvec(x)
    perm = ref.perm()
    b = np.full(N, np.nan)
    for r in range(world):
        rep = h3d.initialize(pts, lap, variant, options=opt, shard_rank=r, shard_world=world)
        st = rep.stats()
        own = perm[st["owned_row_begin"]:st["owned_row_end"]]
        b[own] = rep.matvec(x)[own]
        rep.close()
    assert not np.isnan(b).any()
    assert rel(b, b1) <= 1e-12
    assert rel(b, oracle.dense_matvec(pts, x)) <= 10 * opt.epsilon


@pytest.mark.parametrize("world", [2, 8])
def test_shards_reproduce_single_gpu_clustered(h3d, oracle, world):
    # clustered points: unbalanced Morton subtrees (some shards own few or no
    # rows), empty leaves, leaves above one near pass, cross-shard near pairs
    rng = np.random.default_rng(321)
    centres = rng.uniform(-0.7, 0.7, size=(5, 3))
    n = 8000
    pts = centres[rng.integers(0, 5, n)] + 0.15 * rng.standard_normal((n, 3))
    pts = np.ascontiguousarray(np.clip(pts, -0.999, 0.999))
    x = h3d.random_vector(n, 19)
    # the same explicit representation on every shard (auto scores each
    # shard's own levels and may pick differently from the single-GPU build)
    opt = h3d.HmatOptions(n_max=64, epsilon=1e-7, mode_policy="explicit", level_modes=(0,) + (1,) * 15)
    lap = h3d.make_kernel("laplace3d")
    ref = h3d.initialize(pts, lap, options=opt)
    b1 = ref.matvec(x)
    perm = ref.perm()
    b = np.full(n, np.nan)
    rows_seen = 0
    for r in range(world):
        rep = h3d.initialize(pts, lap, options=opt, shard_rank=r, shard_world=world)
        st = rep.stats()
        own = perm[st["owned_row_begin"]:st["owned_row_end"]]
        rows_seen += len(own)
        if len(own):
            b[own] = rep.matvec(x)[own]
        rep.close()
    assert rows_seen == n and not np.isnan(b).any()
    assert rel(b, b1) <= 1e-12
    assert rel(b, oracle.dense_matvec(pts, x)) <= 10 * opt.epsilon


def test_nccl_exchange_path_world1(h3d):
    # The multi-GPU exchange (own slice of x in Morton order, one NCCL
    # broadcast per rank slice in a group, repack of the source records) run
    # with a 1-rank communicator on one GPU: NCCL resolved by dlopen, the
    # communicator built from a unique id, and the matvec through the
    # exchange path equals the local-gather matvec bit for bit.
    pts = h3d.generate_points(N, SEED)
    x = h3d.random_vector(N, 9)
    opt = h3d.HmatOptions(n_max=64, epsilon=1e-7)
    lap = h3d.make_kernel("laplace3d")
    rep = h3d.initialize(pts, lap, options=opt, shard_rank=0, shard_world=1)
    b0 = rep.matvec(x)
    rep.attach_nccl(h3d.nccl_unique_id(), 0, 1)
    b1 = rep.matvec(x)
    assert np.array_equal(b0, b1)
    led = rep.comm_ledger()
    assert led["x_gather_doubles"] == 0 and led["b_gather_doubles"] == 0 and led["matvecs"] >= 1


def test_nccl_b_allgather_path_world1(h3d):
    # parallel_matvec's full result (parallel.cpp:284-290): with gather_b the
    # owned Morton slices of b are all-gathered after the matvec and the other
    # ranks' rows un-permuted; on a 1-rank communicator the same path runs
    # (broadcast of the one slice + the un-permute pass) and must not change b
    pts = h3d.generate_points(N, SEED)
    x = h3d.random_vector(N, 9)
    lap = h3d.make_kernel("laplace3d")
    ref = h3d.initialize(pts, lap, options=h3d.HmatOptions(n_max=64, epsilon=1e-7)).matvec(x)
    rep = h3d.initialize(pts, lap, options=h3d.HmatOptions(n_max=64, epsilon=1e-7, gather_b=True),
                         shard_rank=0, shard_world=1)
    rep.attach_nccl(h3d.nccl_unique_id(), 0, 1)
    for _ in range(3):
        assert np.array_equal(rep.matvec(x), ref)
    led = rep.comm_ledger()
    assert led["collectives"] == 2 and led["b_gather_doubles"] == 0


def test_gather_b_without_communicator_is_refused(h3d):
    pts = h3d.generate_points(N, SEED)
    rep = h3d.initialize(pts, h3d.make_kernel("laplace3d"),
                         options=h3d.HmatOptions(n_max=64, epsilon=1e-7, gather_b=True),
                         shard_rank=0, shard_world=2)
    with pytest.raises(ValueError):
        rep.matvec(h3d.random_vector(N, 9))


def test_gmres_on_an_attached_shard_world1(h3d):
    # GMRES on a sharded handle: replicated Krylov vectors, every operator
    # application all-gathers b (1-rank communicator here) - the same iterate
    # as the single-GPU solve, bit for bit
    pts = h3d.generate_points(N, SEED)
    lap = h3d.make_kernel("laplace3d")
    opt = h3d.HmatOptions(n_max=64, epsilon=1e-7)
    f = h3d.random_vector(N, 5)
    one = h3d.initialize(pts, lap, options=opt).gmres(f, alpha=2.0, beta=1e-3)
    rep = h3d.initialize(pts, lap, options=opt, shard_rank=0, shard_world=1)
    rep.attach_nccl(h3d.nccl_unique_id(), 0, 1)
    res = rep.gmres(f, alpha=2.0, beta=1e-3)
    assert res.converged and res.iterations == one.iterations
    assert np.array_equal(res.x, one.x)
