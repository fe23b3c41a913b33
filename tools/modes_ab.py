"""Developer probe: device time per matvec over repeated builds of one
configuration, eager launches vs graph replay (H3D_TUNE graphs=0/1), to see
how stable the two-lane co-schedule is.

    python tools/modes_ab.py --builds 3 --steps 20
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_16303_b200 as h3d  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1048576)
    ap.add_argument("--eps", type=float, default=1e-8)
    ap.add_argument("--builds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--tunes", default="graphs=0;graphs=1")
    ap.add_argument("--gap-ms", type=float, default=5.0)
    ap.add_argument("--kernel", default="laplace3d")
    ap.add_argument("--levels", default="auto", help="comma list of auto / explicit level-mode strings")
    a = ap.parse_args()
    import torch
    pts = h3d.generate_points(a.n, 1)
    x = h3d.random_vector(a.n, 18)
    xd = torch.from_numpy(x).cuda()
    bd = torch.empty_like(xd)
    st = torch.cuda.current_stream()
    for lv in a.levels.split(","):
      pol = dict(mode_policy="auto") if lv == "auto" else dict(
          mode_policy="explicit", level_modes=tuple(int(c) for c in lv))
      for tune in a.tunes.split(";"):
        os.environ["H3D_TUNE"] = tune
        for b in range(a.builds):
            rep = h3d.initialize(pts, h3d.make_kernel(a.kernel), "hodlr3d",
                                 h3d.HmatOptions(n_max=64, epsilon=a.eps, **pol))
            for _ in range(3):
                rep.matvec_async(xd.data_ptr(), bd.data_ptr(), st.cuda_stream)
            torch.cuda.synchronize()
            per = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(a.steps):
                    rep.matvec_async(xd.data_ptr(), bd.data_ptr(), st.cuda_stream)
                e1.record(st)
                torch.cuda.synchronize()
                per.append(e0.elapsed_time(e1) / a.steps)
            # the same matvec one at a time, host-synchronised with a gap after each
            single = []
            for _ in range(a.steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                rep.matvec_async(xd.data_ptr(), bd.data_ptr(), st.cuda_stream)
                e1.record(st)
                torch.cuda.synchronize()
                single.append(e0.elapsed_time(e1))
                torch.cuda._sleep(int(a.gap_ms * 1.9e6))
                torch.cuda.synchronize()
            single.sort()
            print(f"levels {lv} tune '{tune}' build {b}: back-to-back ms/matvec " + " ".join(f"{p:.3f}" for p in per) +
                  f" | one at a time (gap {a.gap_ms} ms): median {single[len(single) // 2]:.3f} "
                  f"min {single[0]:.3f}", flush=True)
            rep.close()


if __name__ == "__main__":
    main()
