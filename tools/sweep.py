"""Developer sweep: build once per (level modes, H3D_TUNE) and time the matvec.

    python tools/sweep.py --n 1048576 --eps 1e-8 --levels 011112,011102 --tunes "p2c=2;p2c=3,at=1"
"""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_16303_b200 as h3d  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1048576)
    ap.add_argument("--eps", type=float, default=1e-8)
    ap.add_argument("--kernel", default="laplace3d")
    ap.add_argument("--levels", default="auto")
    ap.add_argument("--tunes", default="")
    ap.add_argument("--reps", type=int, default=6)
    a = ap.parse_args()
    pts = h3d.generate_points(a.n, 1)
    x = h3d.random_vector(a.n, 18)
    for lv in a.levels.split(","):
        for tune in a.tunes.split(";"):
            # eager launches (graphs=0) keep the per-phase timing split
            os.environ["H3D_TUNE"] = ",".join(t for t in ("graphs=0", tune) if t)
            pol = dict(mode_policy="auto") if lv in ("auto", "stream") else dict(
                mode_policy="explicit", level_modes=tuple(int(c) for c in lv))
            if lv == "stream":
                pol = dict(mode_policy="stream")
            t0 = time.time()
            rep = h3d.initialize(pts, h3d.make_kernel(a.kernel), "hodlr3d",
                                 h3d.HmatOptions(n_max=64, epsilon=a.eps, **pol))
            tb = time.time() - t0
            tm = h3d.MatvecTiming()
            rep.matvec(x, timing=tm)
            best = None
            for _ in range(a.reps):
                rep.matvec(x, timing=tm)
                d = tm.gather_ms + tm.exchange_ms + tm.phase1_ms + tm.phase2_ms
                if best is None or d < best[0]:
                    best = (d, tm.phase1_ms, tm.phase2_ms)
            st = rep.stats()
            print(f"levels={lv:8s} modes={''.join(map(str, st['level_modes'][:st['depth'] + 1]))} "
                  f"tune={tune:24s} dev_ms={best[0]:7.3f} p1={best[1]:7.3f} p2={best[2]:7.3f} "
                  f"Mpts/s={a.n / best[0] / 1e3:6.2f} build_s={tb:5.2f} "
                  f"GB={st['factor_doubles'] * 8 / 1e9:6.2f}", flush=True)
            rep.close()
            del rep


if __name__ == "__main__":
    main()
