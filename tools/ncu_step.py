"""Developer driver for ncu captures: build one BASELINE config and run a few
matvecs (eager launches, H3D_TUNE graphs=0 is set here) so a profiler sees
every kernel of a step. Never a bench number.

    ncu --set full -k regex:proxy_solve --launch-count 10 \
        python tools/ncu_step.py --config c3 --matvecs 2
"""
import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("H3D_TUNE", "graphs=0")

from bench import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--matvecs", type=int, default=2)
    ap.add_argument("--policy", default="auto")
    ap.add_argument("--near", default="matrix-free")
    ap.add_argument("--levels", default="", help="explicit level-mode string, e.g. 011142")
    a = ap.parse_args()
    import paper_2307_16303_b200 as h3d
    cfg = CONFIGS[a.config]
    lv = dict(mode_policy=a.policy) if not a.levels else dict(
        mode_policy="explicit", level_modes=tuple(int(c) for c in a.levels))
    pts = h3d.generate_points(cfg["n"], cfg["seed"])
    x = h3d.random_vector(cfg["n"], cfg["seed"] + 17)
    rep = h3d.initialize(pts, h3d.make_kernel(cfg["kernel"]), "hodlr3d",
                         h3d.HmatOptions(n_max=cfg["n_max"], epsilon=cfg["eps"], **lv,
                                         dense_mode="cached" if a.near == "stored" else "on-the-fly"))
    for _ in range(a.matvecs):
        rep.matvec(x)
    st = rep.stats()
    print({k: st[k] for k in ("depth", "level_modes", "build_ms_total", "build_ms_aca_rank",
                              "build_ms_aca_write", "lu_doubles", "factor_doubles", "proxy_units",
                              "level_aca_ms", "level_units")})
    for l in range(1, st["depth"] + 1):
        x, y, r = rep.pairs(l)
        if len(r):
            print(f"level {l}: pairs {len(r)} mean rank {r.mean():.1f} max {r.max()}")


if __name__ == "__main__":
    main()
