"""Developer tool: average board power and energy per matvec for several
representations (nvidia-smi sampled every 20 ms over a long async loop).

    python tools/energy.py --levels stream,011102,011112 [--n 1048576 --eps 1e-8]
"""
import argparse
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402  (before the engine: one libnccl in the process)
import paper_2307_16303_b200 as h3d  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1048576)
    ap.add_argument("--eps", type=float, default=1e-8)
    ap.add_argument("--kernel", default="laplace3d")
    ap.add_argument("--levels", default="auto")
    ap.add_argument("--tunes", default="")
    ap.add_argument("--seconds", type=float, default=3.0)
    a = ap.parse_args()
    pts = h3d.generate_points(a.n, 1)
    x = h3d.random_vector(a.n, 18)
    xd = torch.from_numpy(x).cuda()
    bd = torch.empty_like(xd)
    s = torch.cuda.current_stream().cuda_stream
    for lv in a.levels.split(","):
        for tune in a.tunes.split(";"):
            os.environ["H3D_TUNE"] = tune
            if lv in ("auto", "stream"):
                pol = dict(mode_policy=lv)
            else:
                pol = dict(mode_policy="explicit", level_modes=tuple(int(c) for c in lv))
            rep = h3d.initialize(pts, h3d.make_kernel(a.kernel), "hodlr3d",
                                 h3d.HmatOptions(n_max=64, epsilon=a.eps, **pol))
            for _ in range(3):
                rep.matvec_async(xd.data_ptr(), bd.data_ptr(), s)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                rep.matvec_async(xd.data_ptr(), bd.data_ptr(), s)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            reps = max(20, int(a.seconds * 1e3 / ms))
            log = Path(os.environ.get("TMPDIR", "/tmp")) / "h3d_energy.csv"
            with open(log, "w") as f:
                mon = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm",
                                        "--format=csv,noheader,nounits", "-lms", "20"], stdout=f)
                time.sleep(0.3)
                e0.record()
                for _ in range(reps):
                    rep.matvec_async(xd.data_ptr(), bd.data_ptr(), s)
                e1.record()
                torch.cuda.synchronize()
                time.sleep(0.1)
                mon.terminate()
                mon.wait()
            ms = e0.elapsed_time(e1) / reps
            vals = []
            for line in log.read_text().splitlines():
                try:
                    p, c = (float(v) for v in line.split(","))
                    vals.append((p, c))
                except ValueError:
                    pass
            busy = [v for v in vals if v[0] > 300]
            pw = sum(v[0] for v in busy) / max(len(busy), 1)
            clk = sorted(v[1] for v in busy)[len(busy) // 2] if busy else 0
            st = rep.stats()
            print(f"levels={lv:8s} modes={''.join(map(str, st['level_modes'][:st['depth'] + 1]))} "
                  f"tune={tune:16s} ms={ms:7.3f} avg_W={pw:6.1f} med_sm_MHz={clk:6.0f} "
                  f"J_per_matvec={pw * ms / 1e3:6.2f}", flush=True)
            rep.close()


if __name__ == "__main__":
    main()
