"""Developer probe (needs a -DH3D_DEVTOOLS build, H3D_LIB_PATH): how the two
matvec lanes interfere. For each H3D_TUNE (e.g. skip masks that drop one
lane's kernels) build the configuration once, replay K matvecs back to back
and report ms / matvec, the per-kernel CUDA-event durations of the same
schedule, and the board power / SM clock sampled during the loop.

    H3D_LIB_PATH=tools/lib_dev/libh3d_b200.so python tools/cosched.py \
        --tunes "skip=0;skip=400;skip=10"

Slots (h3d_kernel_slot): 1 p1_stream, 3 p2_stream, 4 p1_proxy, 7 p2_proxy,
8 near. skip=400 = HBM lane only, skip=10 = FP64 lane only. Results with a
skip mask are wrong by construction: timing only.
"""
import argparse
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--tunes", default="skip=0")
    ap.add_argument("--levels", default="auto")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--gap-ms", type=float, default=0.0)
    a = ap.parse_args()
    import torch
    import paper_2307_16303_b200 as h3d
    from bench import CONFIGS
    cfg = CONFIGS[a.config]
    pts = h3d.generate_points(cfg["n"], cfg["seed"])
    x = h3d.random_vector(cfg["n"], cfg["seed"] + 17)
    xd = torch.from_numpy(x).cuda()
    bd = torch.empty_like(xd)
    st = torch.cuda.current_stream()
    names = ["gather", "p1_stream", "red_stream", "p2_stream", "p1_proxy", "red_proxy", "solve",
             "p2_proxy", "near", "combine", "pair", "fused", "half"]
    for lv in a.levels.split(","):
        pol = dict(mode_policy="auto") if lv == "auto" else dict(
            mode_policy="explicit", level_modes=tuple(int(c) for c in lv))
        for tune in a.tunes.split(";"):
            os.environ["H3D_TUNE"] = tune
            rep = h3d.initialize(pts, h3d.make_kernel(cfg["kernel"]), "hodlr3d",
                                 h3d.HmatOptions(n_max=cfg["n_max"], epsilon=cfg["eps"], **pol))
            for _ in range(5):
                rep.matvec_async(xd.data_ptr(), bd.data_ptr(), st.cuda_stream)
            torch.cuda.synchronize()
            log = Path(os.environ.get("TMPDIR", "/tmp")) / "cosched_pow.csv"
            f = open(log, "w")
            mon = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw",
                                    "--format=csv,noheader,nounits", "-lms", "20"], stdout=f)
            time.sleep(0.3)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if a.gap_ms > 0:
                per = []
                for _ in range(a.steps):
                    e0.record(st)
                    rep.matvec_async(xd.data_ptr(), bd.data_ptr(), st.cuda_stream)
                    e1.record(st)
                    torch.cuda.synchronize()
                    per.append(e0.elapsed_time(e1))
                    time.sleep(a.gap_ms * 1e-3)
                ms = statistics.median(per)
            else:
                e0.record(st)
                for _ in range(a.steps):
                    rep.matvec_async(xd.data_ptr(), bd.data_ptr(), st.cuda_stream)
                e1.record(st)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.steps
            mon.terminate()
            mon.wait()
            f.close()
            rows = []
            for line in log.read_text().splitlines():
                p = [s.strip() for s in line.split(",")]
                try:
                    rows.append((float(p[0]), float(p[1]), float(p[2])))
                except (ValueError, IndexError):
                    pass
            rows = rows[len(rows) // 5:]  # drop the ramp
            sm = statistics.median(r[0] for r in rows) if rows else None
            pw = statistics.median(r[2] for r in rows) if rows else None
            pmax = max((r[2] for r in rows), default=None)
            rep.profile(True, 20)
            for _ in range(20):
                rep.matvec_async(xd.data_ptr(), bd.data_ptr(), st.cuda_stream)
            torch.cuda.synchronize()
            rep.profile_read()
            kern = rep.profile_kernels()
            rep.profile(False, 1)
            ks = " ".join(f"{names[k] if isinstance(k, int) else k}={tot / cnt:.2f}@{start / cnt:.2f}"
                          for k, (tot, cnt, start) in kern.items() if cnt)
            print(f"levels={lv} tune={tune:16s} ms={ms:7.3f} Mpts/s={cfg['n'] / ms / 1e3:6.2f} "
                  f"sm_mhz={sm} power_med={pw} power_max={pmax} | {ks}", flush=True)
            rep.close()
            del rep


if __name__ == "__main__":
    main()
