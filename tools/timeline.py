"""Developer tool: per-kernel start/duration timeline of one configuration.

    python tools/timeline.py --levels 011102 [--tune "p1p=2"] [--n 1048576 --eps 1e-8]
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
    ap.add_argument("--kernel", default="laplace3d")
    ap.add_argument("--levels", default="auto")
    ap.add_argument("--tunes", default="")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    pts = h3d.generate_points(a.n, 1)
    x = h3d.random_vector(a.n, 18)
    import torch
    for lv in a.levels.split(","):
        for tune in a.tunes.split(";"):
            os.environ["H3D_TUNE"] = tune
            pol = dict(mode_policy="auto") if lv == "auto" else dict(
                mode_policy="explicit", level_modes=tuple(int(c) for c in lv))
            rep = h3d.initialize(pts, h3d.make_kernel(a.kernel), "hodlr3d",
                                 h3d.HmatOptions(n_max=64, epsilon=a.eps, **pol))
            xd = torch.from_numpy(x).cuda()
            bd = torch.empty_like(xd)
            s = torch.cuda.current_stream().cuda_stream
            for _ in range(3):
                rep.matvec_async(xd.data_ptr(), bd.data_ptr(), s)
            torch.cuda.synchronize()
            rep.profile(True, a.reps)
            for _ in range(a.reps):
                rep.matvec_async(xd.data_ptr(), bd.data_ptr(), s)
            torch.cuda.synchronize()
            prof, n = rep.profile_read()
            kern = rep.profile_kernels()
            st = rep.stats()
            print(f"== levels {lv} modes {st['level_modes'][:st['depth'] + 1]} tune '{tune}' "
                  f"total {prof.total_ms / n:.3f} ms")
            rows = sorted(((v[2] / v[1], v[0] / v[1], k) for k, v in kern.items() if v[1]), key=lambda r: r[0])
            for s0, d, k in rows:
                bar = " " * int(s0 * 2) + "#" * max(1, int(d * 2))
                print(f"  {k:11s} start {s0:7.3f} dur {d:7.3f} end {s0 + d:7.3f} |{bar}")
            rep.close()


if __name__ == "__main__":
    main()
