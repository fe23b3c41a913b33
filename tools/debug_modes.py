"""Developer check: matvec error per representation policy on one config.

    python tools/debug_modes.py --n 4096 --eps 1e-10
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2307_16303_b200 as h3d  # noqa: E402
from oracle_lib import Oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--eps", type=float, default=1e-10)
    ap.add_argument("--nmax", type=int, default=64)
    a = ap.parse_args()
    o = Oracle()
    pts = h3d.generate_points(a.n, 1)
    x = h3d.random_vector(a.n, 18)
    ex = o.dense_matvec(pts, x) if a.n <= 70000 else None
    orep = o.initialize(pts, "laplace3d", n_max=a.nmax, eps=a.eps) if a.n <= 70000 else None
    bo = orep.matvec(x) if orep else None
    L = h3d.initialize(pts, h3d.make_kernel("laplace3d"),
                       options=h3d.HmatOptions(n_max=a.nmax, epsilon=a.eps)).depth
    cfgs = [("stream", ())]
    for l in range(1, L + 1):
        lv = [0] * (L + 1)
        lv[l] = 1
        cfgs.append(("explicit", tuple(lv)))
    cfgs.append(("explicit", tuple([0] * L + [2])))
    cfgs.append(("auto", ()))
    for pol, lv in cfgs:
        rep = h3d.initialize(pts, h3d.make_kernel("laplace3d"),
                             options=h3d.HmatOptions(n_max=a.nmax, epsilon=a.eps, mode_policy=pol,
                                                     level_modes=lv))
        b = rep.matvec(x)
        st = rep.stats()
        msg = f"{pol:9s} {str(lv):20s} modes {st['level_modes']}"
        if ex is not None:
            msg += f" err_exact {np.linalg.norm(b - ex) / np.linalg.norm(ex):.3e}"
            msg += f" vs_oracle {np.linalg.norm(b - bo) / np.linalg.norm(bo):.3e}"
        print(msg, flush=True)
        rep.close()


if __name__ == "__main__":
    main()
