"""Golden fixtures at the BASELINE sizes, from the REFERENCE ITSELF
(oracle/_ref). Long-running (the reference initialize takes ~6 min at N=1M on
8 cores), so only small per-config summaries are stored:

* a digest (SHA-256) of the tree and lists: perm, every level's offsets and
  interaction lists,
* the reference matvec b_ref and the exact sum b_exact on 2000 rows drawn by
  reference_error's rule (mt19937_64(7), hmatrix.cpp:263-266), plus the
  reference's own reference_error value,
* per-level rank summaries (count, sum, max of the ordered block ranks),
* the reference's full matvec output b_ref (every config up to C3: 8 MB),
* C5 (N = 4,194,304): the tree/list digest only (the reference's
  build_tree + build_interaction_lists; its initialize would need ~66 GB).

    python tests/golden/make_golden_large.py c2 c4 c3 c5
"""
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import Oracle, RefLib  # noqa: E402

CONFIGS = {
    "c2": (65536, "laplace3d", 64, 1e-10, 1),
    "c3": (1048576, "laplace3d", 64, 1e-8, 1),
    "c4": (262144, "r4", 64, 1e-8, 1),
    "c5": (4194304, "laplace3d", 64, 1e-6, 1),  # tree / lists only
}
TREE_ONLY = {"c5"}


def tree_digest(rep):
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


def sample_rows(n, count=2000, seed=7):
    u = Oracle().uniform_stream(count, seed)
    return (u * n).astype(np.int64)  # permuted positions (hmatrix.cpp:263-266)


def main(names):
    ref = RefLib()
    ref.set_threads(8)
    o = Oracle()
    o.set_threads(8)
    for name in names:
        n, kern, n_max, eps, seed = CONFIGS[name]
        pts = ref.generate_points(n, seed)
        x = ref.random_vector(n, seed + 17)
        if name in TREE_ONLY:
            t0 = time.time()
            rep = ref.tree_lists(pts, n_max=n_max)
            out = dict(n=n, kernel=kern, n_max=n_max, eps=eps, seed=seed, depth=rep.depth,
                       tree_digest=tree_digest(rep), tree_only=True)
            np.savez_compressed(HERE / f"large_{name}.npz", **out)
            print(name, "depth", rep.depth, "tree+lists", round(time.time() - t0, 1), "s", flush=True)
            continue
        t0 = time.time()
        rep = ref.initialize(pts, kern, n_max=n_max, eps=eps)
        t1 = time.time()
        b = rep.matvec(x)
        ref_err = rep.reference_error(x, b)
        perm = rep.perm()
        rows = perm[sample_rows(n)].astype(np.int64)  # original indices of the sampled rows
        ex = o.exact_rows(pts, x, rows, kern)
        ranks = []
        for l in range(1, rep.depth + 1):
            _, _, r = rep.lr_blocks(l)
            ranks.append([l, len(r), int(r.sum()), int(r.max()) if len(r) else 0])
        out = dict(n=n, kernel=kern, n_max=n_max, eps=eps, seed=seed, depth=rep.depth,
                   tree_digest=tree_digest(rep), rows=rows, b_ref_rows=b[rows],
                   b_exact_rows=ex, ref_error=ref_err, ranks=np.array(ranks, dtype=np.int64),
                   ref_init_s=t1 - t0)
        out["b_ref"] = b
        np.savez_compressed(HERE / f"large_{name}.npz", **out)
        print(name, "depth", rep.depth, "init", round(t1 - t0, 1), "ref_error", ref_err,
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c4", "c3", "c5"])
