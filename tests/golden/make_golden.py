"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Runs the unmodified reference (oracle/_ref/libh3dref.so, built in place from
/root/reference/proj/src by `make -C oracle ref`) on seeded inputs and stores
its outputs: permutation, node offsets, interaction lists, per-block ranks,
its matvec output b_ref and the exact direct sum b_exact.

Only runnable where /root/reference was mounted at build time; the fixtures
are committed so the GPU box (no /root/reference) can use them.

    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import RefLib  # noqa: E402

# name: (N, kernel, n_max, eps, seed[, variant[, {diag, max_rank}]])  -- C1 is
# BASELINE.json configs[0]; the last two exercise HmatOptions::max_rank
# (hmatrix.hpp:21, lowrank.cpp rank cap) and KernelSpec::diagonal (kernel.hpp:49)
CONFIGS = {
    # the other two block structures of the reference (octree.cpp:197-260)
    "hodlr_n3000_laplace_nmax100_eps1e-6": (3000, "laplace3d", 100, 1e-6, 29, "hodlr"),
    "hodlr_n12000_r4_nmax64_eps1e-8": (12000, "r4", 64, 1e-8, 41, "hodlr"),
    "hstrong_n3000_helm_nmax100_eps1e-6": (3000, "helmholtz-re", 100, 1e-6, 29, "hstrong"),
    "hstrong_n20000_laplace_nmax64_eps1e-8": (20000, "laplace3d", 64, 1e-8, 43, "hstrong"),
    "c1_n4096_laplace_nmax64_eps1e-10": (4096, "laplace3d", 64, 1e-10, 1),
    "n3000_r4_nmax100_eps1e-6": (3000, "r4", 100, 1e-6, 29),
    "n3000_helm_nmax100_eps1e-6": (3000, "helmholtz-re", 100, 1e-6, 29),
    "n150_laplace_depth0": (150, "laplace3d", 216, 1e-7, 19),
    "n2197_laplace_nmax64_eps1e-7": (2197, "laplace3d", 64, 1e-7, 13),
    "n3000_laplace_nmax64_eps1e-8_maxrank12": (3000, "laplace3d", 64, 1e-8, 47, "hodlr3d",
                                                {"max_rank": 12}),
    "n5000_r4_nmax100_eps1e-7_diag2.5": (5000, "r4", 100, 1e-7, 53, "hodlr3d", {"diag": 2.5}),
}


def main(only=()):
    ref = RefLib()
    ref.set_threads(8)
    for name, cfg in CONFIGS.items():
        if only and name not in only:
            continue
        n, kern, n_max, eps, seed = cfg[:5]
        variant = cfg[5] if len(cfg) > 5 else "hodlr3d"
        extra = cfg[6] if len(cfg) > 6 else {}
        diag, max_rank = float(extra.get("diag", 0.0)), int(extra.get("max_rank", 0))
        pts = ref.generate_points(n, seed)
        x = ref.random_vector(n, seed + 17)
        rep = ref.initialize(pts, kern, n_max=n_max, eps=eps, variant=variant, diag=diag,
                             max_rank=max_rank)
        out = dict(n=n, kernel=kern, n_max=n_max, eps=eps, seed=seed, depth=rep.depth,
                   perm=rep.perm(), x=x, variant=variant, diag=diag, max_rank=max_rank)
        for l in range(rep.depth + 1):
            out[f"off{l}"] = rep.offsets(l)
            for k, kn in enumerate(["inter", "edge", "face", "vertex"]):
                o, ids = rep.list(l, k)
                out[f"{kn}_off{l}"] = o
                out[f"{kn}_ids{l}"] = ids
            if l >= 1:
                t, s, r = rep.lr_blocks(l)
                out[f"lr_t{l}"], out[f"lr_s{l}"], out[f"lr_r{l}"] = t, s, r
        out["b_ref"] = rep.matvec(x)
        out["b_exact"] = ref.dense_matvec(pts, x, kern, diag)
        out["ref_error"] = rep.reference_error(x, out["b_ref"])
        st = rep.stats()
        out["stats"] = np.array([st["float_count"], st["int_count"], st["memory_bytes"],
                                 st["max_rank"], st["depth"]], dtype=np.uint64)
        np.savez_compressed(HERE / f"{name}.npz", **out)
        print(name, "depth", rep.depth, "err", out["ref_error"])


if __name__ == "__main__":
    main(tuple(sys.argv[1:]))
