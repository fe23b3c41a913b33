"""Developer probe: build + time a configuration on the GPU and print stats.

    python tools/probe.py --n 65536 --eps 1e-10 --nmax 64 [--kernel r4] [--mode cached]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_16303_b200 as h3d  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--eps", type=float, default=1e-10)
    ap.add_argument("--nmax", type=int, default=64)
    ap.add_argument("--kernel", default="laplace3d")
    ap.add_argument("--mode", default="on-the-fly")
    ap.add_argument("--policy", default="auto")
    ap.add_argument("--levels", default="")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check-rows", type=int, default=0)
    a = ap.parse_args()
    os.environ.setdefault("H3D_TUNE", "graphs=0")  # eager: keeps the per-phase timing split
    t0 = time.time()
    pts = h3d.generate_points(a.n, a.seed)
    x = h3d.random_vector(a.n, a.seed + 17)
    t1 = time.time()
    rep = h3d.initialize(pts, h3d.make_kernel(a.kernel), "hodlr3d",
                         h3d.HmatOptions(n_max=a.nmax, epsilon=a.eps, dense_mode=a.mode,
                                         mode_policy=a.policy,
                                         level_modes=tuple(int(c) for c in a.levels)))
    t2 = time.time()
    st = rep.stats()
    tm = h3d.MatvecTiming()
    b = rep.matvec(x, timing=tm)
    times = []
    for _ in range(a.reps):
        rep.matvec(x, timing=tm)
        times.append(dict(tm.__dict__))
    best = min(times, key=lambda d: d["total_ms"])
    out = dict(n=a.n, eps=a.eps, kernel=a.kernel, mode=a.mode, gen_s=t1 - t0, build_s=t2 - t1,
               stats=st, best=best,
               mpts_host=a.n / best["total_ms"] / 1e3,
               mpts_dev=a.n / (best["phase1_ms"] + best["phase2_ms"] + best["gather_ms"]) / 1e3,
               factor_GB=st["factor_doubles"] * 8 / 1e9)
    p1 = best["phase1_ms"]
    p2 = best["phase2_ms"]
    out["phase1_GBs"] = st["factor_doubles"] * 8 / 1e6 / p1 if p1 > 0 else 0
    out["phase2_GBs"] = st["factor_doubles"] * 8 / 1e6 / p2 if p2 > 0 else 0
    if a.check_rows:
        sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
        from oracle_lib import Oracle
        o = Oracle()
        rng = np.random.default_rng(0)
        rows = rng.integers(0, a.n, a.check_rows)
        ex = o.exact_rows(pts, x, rows, a.kernel)
        out["sampled_err"] = float(np.linalg.norm(b[rows] - ex) / np.linalg.norm(ex))
    print(json.dumps(out, indent=1, default=float))


if __name__ == "__main__":
    main()
