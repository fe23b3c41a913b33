"""Developer stress loop: repeat build + matvec on one golden case and report
hangs / mismatches per H3D_TUNE setting (each setting in its own process
under a wall-clock limit, with a faulthandler dump when a call stalls).

    python tools/stress.py --case hodlr_n12000_r4_nmax64_eps1e-8 --reps 50 \
        --tunes "fw=1" "fw=0" "graphs=0" --mode cached
"""
import argparse
import faulthandler
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def child(a):
    sys.path.insert(0, str(ROOT))
    import paper_2307_16303_b200 as h3d
    with np.load(ROOT / "tests" / "golden" / f"{a.case}.npz") as z:
        g = {k: z[k] for k in z.files}
    n, seed, eps = int(g["n"]), int(g["seed"]), float(g["eps"])
    pts = h3d.generate_points(n, seed)
    variant = str(g.get("variant", "hodlr3d"))
    bref = g["b_ref"]
    worst = 0.0
    t0 = time.time()
    for i in range(a.reps):
        faulthandler.dump_traceback_later(a.stall, exit=True)
        rep = h3d.initialize(pts, h3d.make_kernel(str(g["kernel"])), variant,
                             h3d.HmatOptions(n_max=int(g["n_max"]), epsilon=eps, dense_mode=a.mode,
                                             mode_policy=a.policy))
        for k in range(a.matvecs):
            b = rep.matvec(g["x"])
            e = float(np.linalg.norm(b - bref) / np.linalg.norm(bref))
            worst = max(worst, e)
            if e > 10 * eps:
                print(json.dumps({"rep": i, "matvec": k, "rel": e, "bad": True}), flush=True)
        rep.close()
        faulthandler.cancel_dump_traceback_later()
    print(json.dumps({"reps": a.reps, "worst_rel": worst, "s": round(time.time() - t0, 2)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="hodlr_n12000_r4_nmax64_eps1e-8")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--matvecs", type=int, default=4)
    ap.add_argument("--mode", default="cached")
    ap.add_argument("--policy", default="auto")
    ap.add_argument("--stall", type=float, default=30.0)
    ap.add_argument("--limit", type=float, default=300.0)
    ap.add_argument("--tunes", nargs="*", default=[""])
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a)
        return
    for tune in a.tunes:
        env = dict(os.environ, H3D_TUNE=tune)
        cmd = [sys.executable, __file__, "--child", "--case", a.case, "--reps", str(a.reps),
               "--matvecs", str(a.matvecs), "--mode", a.mode, "--policy", a.policy,
               "--stall", str(a.stall)]
        t0 = time.time()
        try:
            r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=a.limit)
            rc, out, err = r.returncode, r.stdout, r.stderr
        except subprocess.TimeoutExpired as e:
            rc, out, err = "timeout", (e.stdout or b"").decode() if isinstance(e.stdout, bytes) else (e.stdout or ""), \
                (e.stderr or b"").decode() if isinstance(e.stderr, bytes) else (e.stderr or "")
        print(f"== tune={tune!r} mode={a.mode} policy={a.policy} rc={rc} {time.time() - t0:.1f}s", flush=True)
        print(out.strip()[-2000:], flush=True)
        if rc != 0:
            print(err.strip()[-4000:], flush=True)


if __name__ == "__main__":
    main()
