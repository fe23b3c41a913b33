"""Developer probe: build-time breakdown of one BASELINE config (repeated
builds; the first includes lazy module loading).

    python tools/build_probe.py --config c3 --builds 3
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--builds", type=int, default=3)
    ap.add_argument("--tunes", default="", help="';'-separated H3D_TUNE values, one build series each")
    a = ap.parse_args()
    import paper_2307_16303_b200 as h3d
    from bench import CONFIGS
    cfg = CONFIGS[a.config]
    pts = h3d.generate_points(cfg["n"], cfg["seed"])
    import os
    for tune in a.tunes.split(";"):
      os.environ["H3D_TUNE"] = tune
      print(f"H3D_TUNE={tune}", flush=True)
      for b in range(a.builds):
        t0 = time.time()
        rep = h3d.initialize(pts, h3d.make_kernel(cfg["kernel"]), "hodlr3d",
                             h3d.HmatOptions(n_max=cfg["n_max"], epsilon=cfg["eps"]))
        wall = time.time() - t0
        st = rep.stats()
        keys = ["build_ms_tree", "build_ms_lists", "build_ms_aca_rank", "build_ms_plan", "build_ms_aca_write",
                "build_ms_post", "build_ms_near", "build_ms_total"]
        print(f"build {b}: wall {wall * 1e3:.0f} ms | " + " ".join(f"{k[9:]}={st[k]:.0f}" for k in keys) +
              " | level_aca_ms " + " ".join(f"{v:.0f}" for v in st["level_aca_ms"][1:st["depth"] + 1]) +
              f" | sum_rank {st['sum_rank']}", flush=True)
        rep.close()


if __name__ == "__main__":
    main()
