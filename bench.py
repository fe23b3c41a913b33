#!/usr/bin/env python
"""HODLR3D matvec benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3] [--near matrix-free|stored]

One step = one full HODLR3D matvec b = A~ x of the BASELINE workload
(configs[2], "C3": N = 1,048,576 uniform points, Laplace 1/r, diag 0, fp64,
leaf n_max = 64, ACA tol 1e-8, single RHS) with x and b resident in HBM.
Multi-GPU (torchrun, one rank per GPU): Morton-subtree row ownership, the x
all-gather over NVLink inside the step; the time is the max over ranks.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libh3dref.so, the unmodified sources compiled in place) on all
of the box's host cores on the SAME workload (N, kernel, tol, n_max, inputs):
initialize once (untimed, reported), then W warm-up and K timed matvecs.
The `cpu_baseline` of our own arm is a bounded sample (N = 262,144, a few
matvecs) so the default run stays short; the headline CPU comparison is the
reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "HODLR3D matvec Mpoints/s at N=1M Laplace (1/2/4/8 GPU); % of HBM roofline"

CONFIGS = {
    "c1": dict(n=4096, kernel="laplace3d", eps=1e-10, n_max=64, seed=1,
               desc="C1: N=4,096 uniform [-1,1]^3, Laplace 1/r (diag 0), fp64, n_max 64, ACA tol 1e-10"),
    "c2": dict(n=65536, kernel="laplace3d", eps=1e-10, n_max=64, seed=1,
               desc="C2: N=65,536 uniform [-1,1]^3, Laplace 1/r (diag 0), fp64, n_max 64, ACA tol 1e-10"),
    "c3": dict(n=1048576, kernel="laplace3d", eps=1e-8, n_max=64, seed=1,
               desc="C3: N=1,048,576 uniform [-1,1]^3, Laplace 1/r (diag 0), fp64, n_max 64, "
                    "ACA tol 1e-8, single RHS x~U[-1,1]"),
    "c4": dict(n=262144, kernel="r4", eps=1e-8, n_max=64, seed=1,
               desc="C4: N=262,144 uniform [-1,1]^3, 1/r^4 (diag 0), fp64, n_max 64, ACA tol 1e-8"),
    "c5": dict(n=4194304, kernel="laplace3d", eps=1e-6, n_max=64, seed=1,
               desc="C5: N=4,194,304 uniform [-1,1]^3, Laplace 1/r (diag 0), fp64, n_max 64, "
                    "ACA tol 1e-6, matrix-free near field"),
}
# cpu_baseline sample size of our own arm (the CPU reference needs ~6 min per
# initialize at N=1M on 8 cores), same generator /
# kernel / tol / n_max. The reference arm (--impl reference) runs the full N.
REF_SAMPLE_N = {"c1": 4096, "c2": 65536, "c3": 262144, "c4": 65536, "c5": 262144}

FALLBACK_HBM = 6650.0  # GB/s, /opt/skills/guides/B200_PROFILING.md fallback
# FP64 peak is not in MEASURED_PEAKS.json; measured on this pool's B200 with
# tools/fp64_bench.cu: 17.49 T DFMA/s sustained = 35.0 TFLOP/s (profiles/r01_summary.md).
# The FP64 roofline counts FP64-pipe instructions (DADD/DMUL/DFMA all issue at
# the DFMA rate) and reports them FMA-equivalent: achieved TFLOP/s = 2 x
# instructions/s, peak 35.0.
FP64_INSTR_PEAK = 17.49e12
FP64_TFLOPS = 2 * FP64_INSTR_PEAK / 1e12
# FP64-pipe instructions per kernel evaluation (SASS of the matvec kernels):
# r^2 = 3 DADD + DMUL + 2 DFMA; Laplace admissible (Newton form) 4 more,
# dense-near (third-order rsqrt) 6 more; 1/r^4 and cos(r)/r use the exact
# radial maps (reciprocal / sincos sequences).
INSTR_FAR = {"laplace3d": 10, "r4": 12, "helmholtz-re": 40}
# What the register file lets the Laplace admissible core reach: a DFMA with
# three distinct register operands takes 3 cycles per sub-partition, not 2
# (one 64-bit operand read per cycle), and a broadcast LDS.128 ~1.4; the
# kernels' loop (2 targets x 4 sources per trip, 18.0-18.6 operand reads + 1.5
# LDS.128 per evaluation) runs at 1.76 T evaluations/s in isolation
# (tools/eval_bench.cu, profiles/r02_eval_bench.log, profiles/r02_summary.md).
CORE_EVALS_PER_S = {"laplace3d": 1.76e12}
# half levels' regenerated side (matvec.cu half2_kernel): one evaluation (the
# far value without the accumulate) feeding two FMAs, plus ~0.6 DADD of the
# 8-source warp reduce-scatter per entry
INSTR_HALF = {"laplace3d": 10, "r4": 12, "helmholtz-re": 42}
INSTR_NEAR = {"laplace3d": 12, "r4": 14, "helmholtz-re": 40}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"h3d_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.f.close()
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [s.strip() for s in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append(dict(sm=float(parts[1]), smax=float(parts[2]), power=float(parts[3]),
                                 hw=parts[5], hwth=parts[6], swth=parts[7], swpc=parts[8]))
            except ValueError:
                continue
        try:
            self.path.unlink()
        except OSError:
            pass
        if not rows:
            return None
        reasons = set()
        for r in rows:
            for key, name in [("hw", "hw_slowdown"), ("hwth", "hw_thermal_slowdown"),
                              ("swth", "sw_thermal_slowdown"), ("swpc", "sw_power_cap")]:
                if r[key].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in rows), "sm_max_mhz": rows[0]["smax"],
                "reasons": sorted(reasons), "samples": len(rows),
                "power_w_max": max(r["power"] for r in rows),
                "power_w_median": statistics.median(r["power"] for r in rows)}


# ------------------------------------------------------------------ CPU baseline
def workload_config(cfg_name: str, near: str) -> dict:
    """The `config` object both arms print (identical, so the driver can pair
    them); diagnostics go to the line's `detail`."""
    cfg = CONFIGS[cfg_name]
    return {"workload": cfg["desc"], "n": cfg["n"], "kernel": cfg["kernel"], "aca_tol": cfg["eps"],
            "n_max": cfg["n_max"], "variant": "hodlr3d",
            "near_field": "on-the-fly (DenseMode::OnTheFly, matrix-free)" if near == "matrix-free"
                          else "cached (DenseMode::Cached, stored)",
            "inputs": "generate_points(UniformRandom, N, seed=1); x = 2u-1 from mt19937_64(18)",
            "l2": "no flush: every step streams a working set far larger than the 126 MB L2 "
                  "(GPU: factor pool + LU + points, tens of GB at C3; CPU: the reference's "
                  "block list)"}


def reference_cpu_run(cfg_name: str, steps: int, warmup: int, n: int | None = None,
                      near: str = "matrix-free"):
    """Time the reference CPU matvec (oracle/_ref) on all host cores; n=None:
    the workload's own N, else a bounded sample of that size."""
    from oracle_lib import REF_REL_SO, RefLib, have_ref, host_has_avx512
    build = "pinned parity build (-O3 -march=x86-64-v3 -ffp-contract=off)"
    if not have_ref():
        from oracle_lib import Oracle
        lib, kind = Oracle(), "port"
        build = "C restatement oracle/h3d_oracle.c"
    elif REF_REL_SO.exists() and host_has_avx512():
        # the reference's release flags (proj/CMakeLists.txt:17: -O3 -march=native
        # -fno-math-errno) for this AVX-512 host
        lib, kind = RefLib(REF_REL_SO), "reference"
        build = "release build (-O3 -march=x86-64-v4 -fno-math-errno, FP contraction on)"
    else:
        lib, kind = RefLib(), "reference"
    cores = os.cpu_count() or 1
    lib.set_threads(cores)
    cfg = CONFIGS[cfg_name]
    full = n is None
    n = cfg["n"] if full else n
    pts = lib.generate_points(n, cfg["seed"])
    x = lib.random_vector(n, cfg["seed"] + 17)
    t0 = time.time()
    kw = {"cached": near == "stored"} if kind == "reference" else {}
    rep = lib.initialize(pts, cfg["kernel"], n_max=cfg["n_max"], eps=cfg["eps"], **kw)
    init_s = time.time() - t0
    for _ in range(warmup):
        rep.matvec(x)
    ts = []
    for _ in range(steps):
        t1 = time.perf_counter()
        rep.matvec(x)
        ts.append(time.perf_counter() - t1)
    mean = sum(ts) / len(ts)
    model = "unknown CPU"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    what = ("the full workload" if full else
            "a bounded sample (smaller N than the workload favours the reference: its per-point "
            "cost grows with N)")
    return dict(value=n / mean / 1e6, unit="Mpoints/s", cores=cores, kind=kind,
                sample=(f"reference matvec (hmatrix.cpp:153-226, OpenMP {cores} threads on {model}) at N={n}, "
                        f"{what} (same generator/kernel/tol/n_max, depth {rep.depth}); "
                        f"mean of {steps} steps after {warmup} warm-up; initialize {init_s:.1f} s untimed"),
                init_s=init_s, ms_per_step=mean * 1e3, n=n, cpu_model=model, depth=rep.depth, build=build)


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--near", default="matrix-free", choices=["matrix-free", "stored"])
    ap.add_argument("--policy", default="auto", choices=["auto", "stream"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        r = reference_cpu_run(args.config, args.steps, args.warmup, near=args.near)
        line = {"metric": METRIC, "value": r["value"], "unit": "Mpoints/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic: generate_points(UniformRandom, N, seed=1) and x = 2u-1 from "
                        "mt19937_64(18), the reference's own generators",
                "config": workload_config(args.config, args.near),
                "detail": {"n": r["n"], "depth": r["depth"], "initialize_s": round(r["init_s"], 2),
                           "threads": r["cores"], "cpu_model": r["cpu_model"],
                           "build": "oracle/Makefile: unmodified /root/reference/proj/src compiled "
                                    "in place with OpenMP against the Eigen/doctest API shims, "
                                    + r["build"]},
                "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": r["value"], "unit": "Mpoints/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import numpy as np
    import torch
    import paper_2307_16303_b200 as h3d

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    n = cfg["n"]
    pts = h3d.generate_points(n, cfg["seed"])
    x_host = h3d.random_vector(n, cfg["seed"] + 17)
    opt = h3d.HmatOptions(n_max=cfg["n_max"], epsilon=cfg["eps"],
                          dense_mode="cached" if args.near == "stored" else "on-the-fly",
                          mode_policy=args.policy)
    # process warm-up (lazy module loading, allocator): a small build first, so
    # aca_build_s is the workload's own build
    h3d.initialize(h3d.generate_points(20000, 3), h3d.make_kernel(cfg["kernel"]), "hodlr3d",
                   h3d.HmatOptions(n_max=cfg["n_max"], epsilon=cfg["eps"]), device=local_rank).close()
    t0 = time.time()
    rep = h3d.initialize(pts, h3d.make_kernel(cfg["kernel"]), "hodlr3d", opt, device=local_rank,
                         shard_rank=rank, shard_world=world)
    build_s = time.time() - t0
    if world > 1:
        uid = [h3d.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        rep.attach_nccl(uid[0], rank, world)
    st = rep.stats()

    dev = torch.device("cuda", local_rank)
    x = torch.from_numpy(x_host).to(dev)
    b = torch.empty(n, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    # warm-up (untimed)
    for _ in range(args.warmup):
        rep.matvec_async(x.data_ptr(), b.data_ptr(), sp)
    torch.cuda.synchronize(dev)

    # ---- timed region: K device-resident steps, CUDA events on the launch stream
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        rep.matvec_async(x.data_ptr(), b.data_ptr(), sp)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_local = ms
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n / (ms * 1e-3) / 1e6

    # ---- per-kernel durations: the same K steps again with a CUDA-event pair
    # around every kernel on its own lane (untimed for the headline number)
    rep.profile(True, args.steps)
    for _ in range(args.steps):
        rep.matvec_async(x.data_ptr(), b.data_ptr(), sp)
    torch.cuda.synchronize(dev)
    prof, nprof = rep.profile_read()
    kern = rep.profile_kernels()
    rep.profile(False, 1)

    # ---- e2e: the public C-ABI call with pinned host buffers (H2D x, D2H b)
    xh = torch.from_numpy(x_host.copy()).pin_memory()
    bh = torch.empty(n, dtype=torch.float64).pin_memory()
    for _ in range(2):
        rep.matvec_ptr(xh.data_ptr(), bh.data_ptr(), host=True)
    if dist:
        dist.barrier()
    t_e2e, t_h2d, t_d2h = [], [], []
    tm = h3d.MatvecTiming()
    for _ in range(args.steps):
        rep.matvec_ptr(xh.data_ptr(), bh.data_ptr(), host=True, timing=tm)
        t_e2e.append(tm.total_ms)
        t_h2d.append(tm.h2d_ms)
        t_d2h.append(tm.d2h_ms)
    e2e_ms = sum(t_e2e) / len(t_e2e)
    if dist:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = n / (e2e_ms * 1e-3) / 1e6

    # ---- per-rank work (multi-GPU): owned rows, streamed bytes, regenerated
    # entries and device time of each shard (balance check)
    per_rank = None
    if dist:
        try:
            mine = {"rank": rank, "owned_rows": int(st["owned_row_end"] - st["owned_row_begin"]),
                    "streamed_factor_GB_per_phase": round(8 * st["factor_doubles"] / 1e9, 3),
                    "proxy_entries_per_phase": int(st["proxy_units"]), "ms_per_step": round(ms_local, 4)}
            per_rank = [None] * world
            dist.all_gather_object(per_rank, mine)
        except Exception as e:  # reporting only
            per_rank = f"unavailable: {e}"

    # ---- parity spot check on 200 sampled rows against the exact sum (oracle)
    rel_err = None
    if rank == 0:
        try:
            from oracle_lib import Oracle
            o = Oracle()
            o.set_threads(os.cpu_count() or 1)
            rows = np.random.default_rng(7).integers(0, n, 200)
            bb = bh.numpy()
            own = rep.perm()[st["owned_row_begin"]:st["owned_row_end"]]
            mask = np.isin(rows, own)
            if mask.any():
                ex = o.exact_rows(pts, x_host, rows[mask], cfg["kernel"])
                rel_err = float(np.linalg.norm(bb[rows[mask]] - ex) / np.linalg.norm(ex))
        except Exception as e:  # checker unavailable: report, never substitute
            rel_err = f"unavailable: {e}"

    # ---- roofline. Algorithmic work per launch of each kernel (DESIGN.md
    # section 6): stream kernels = the streamed factor bytes of one phase;
    # proxy kernels = one phase's regenerated entries x FP64 instructions per
    # entry; near pass = dense-near + direct entries; solves = both
    # orientations' triangular inverses. Dominant kernel = largest mean
    # CUDA-event duration (lanes overlap, so shares are of the summed kernel time).
    hbm, peak_src = peaks()
    F = st["factor_doubles"]           # streamed factor doubles per phase (stream levels)
    HU = st["half_units"]              # half levels: regenerated entries, evaluated once for both phases
    U = st["proxy_units"] - HU         # regenerated entries per phase (proxy levels)
    NEAR, DIRECT = st["near_entries"], st["direct_evals"]
    LU = st["lu_doubles"]
    kf, kn = INSTR_FAR[cfg["kernel"]], INSTR_NEAR[cfg["kernel"]]
    nlev = sum(1 for m in st["level_modes"][1:st["depth"] + 1] if m in (0, 1))
    work = {
        "p1_stream": ("hbm", 8.0 * F), "p2_stream": ("hbm", 8.0 * F),
        "p1_proxy": ("fp64", kf * U), "p2_proxy": ("fp64", kf * U),
        "near": ("fp64", kn * NEAR + kf * DIRECT), "solve": ("hbm", 2 * 8.0 * LU),
        "gather": ("hbm", 8.0 * (4 * n)), "combine": ("hbm", 8.0 * n * (2 + nlev)),
        "red_stream": ("hbm", 0.0), "red_proxy": ("hbm", 0.0),
        "half": ("fp64", INSTR_HALF[cfg["kernel"]] * HU),
    }
    kstats = {}
    for k, (tot, cnt, start) in kern.items():
        if cnt == 0:
            continue
        kms = tot / cnt
        bound, w = work[k]
        if bound == "hbm":
            ach, pk, unit = w / (kms * 1e-3) / 1e9, hbm, "GB/s"
        else:
            ach, pk, unit = 2 * w / (kms * 1e-3) / 1e12, FP64_TFLOPS, "TFLOP/s"
        kstats[k] = dict(ms=round(kms, 4), start_ms=round(start / cnt, 4), bound=bound,
                         achieved=round(ach, 3), peak=pk, unit=unit, frac=round(ach / pk, 4))
        if k in ("p1_proxy", "p2_proxy") and cfg["kernel"] in CORE_EVALS_PER_S and U > 0:
            # the same kernel against the operand-read bound of its evaluation core
            ev = U / (kms * 1e-3)
            kstats[k]["evals_per_s"] = round(ev / 1e12, 4)
            kstats[k]["frac_of_operand_bound"] = round(ev / CORE_EVALS_PER_S[cfg["kernel"]], 4)
    ksum = sum(v["ms"] for v in kstats.values())
    for v in kstats.values():
        v["share"] = round(v["ms"] / ksum, 4) if ksum else None
    dom = max(kstats, key=lambda k: kstats[k]["ms"])
    kd = kstats[dom]
    traffic = None
    tr = ROOT / "profiles" / "ncu_traffic.json"
    if tr.exists():
        try:
            d = json.loads(tr.read_text())
            if d.get("config") == args.config and d.get("level_modes") == st["level_modes"][:st["depth"] + 1]:
                traffic = d.get("kernels", {}).get(dom)
        except Exception:
            traffic = None
    # step roofline: both resources busy the whole step at best
    step_bytes = sum(work[k][1] for k in kstats if work[k][0] == "hbm")
    step_instr = sum(work[k][1] for k in kstats if work[k][0] == "fp64")
    t_hbm = step_bytes / (hbm * 1e9) * 1e3
    t_fp = step_instr / FP64_INSTR_PEAK * 1e3
    step_roof_ms = max(t_hbm, t_fp)
    # the factor-streaming representation's HBM roofline (what the reference's
    # matvec would need on this GPU): every level's factors read in both
    # phases + the stored dense near field (leaf-level admissible blocks that
    # we evaluate directly are left out: a lower bound)
    units_all = sum(st["level_units"][1:st["depth"] + 1])
    stream_repr_bytes = 2 * 8.0 * units_all + 8.0 * NEAR + 16.0 * n
    t_stream_repr = stream_repr_bytes / (hbm * 1e9) * 1e3

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        r = reference_cpu_run(args.config, steps=3, warmup=1, n=REF_SAMPLE_N[args.config])
        cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "Mpoints/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: generate_points(UniformRandom, N, seed=1) and x = 2u-1 from "
                "mt19937_64(18), bit-identical to the reference generators",
        "config": workload_config(args.config, args.near),
        "detail": {
            "representation": {"policy": args.policy,
                               "level_modes": {str(l): ["stream", "proxy", "direct", "pair", "fused", "half", "split"][m]
                                               for l, m in enumerate(st["level_modes"]) if l > 0},
                               "note": "one ACA per unordered admissible pair; stream = explicit "
                                       "factors in HBM, proxy = pivots+LU regenerated in FP64, "
                                       "half = U' = K(X,tau)(LR)^-1 streamed + K(sigma,Y) "
                                       "regenerated (no solves), direct = exact leaf blocks"},
            "streamed_factor_GB_per_phase": round(8 * F / 1e9, 3),
            "proxy_entries_per_phase": U,
            "lu_GB": round(8 * st["lu_doubles"] / 1e9, 3),
            "parallelism": f"Morton-subtree row ownership over {world} GPU(s), NCCL all-gather of x",
            "l2": f"inputs larger than L2: per-step working set (factor pool, LU inverses, proxy "
                  f"points/t-vectors, packed points) "
                  f"{8 * (st['factor_bytes_alloc'] / 8 + 2 * LU + 4 * st['tvec_doubles'] + 5 * n) / 1e9:.2f} GB "
                  f">> 126 MB L2",
            "aca_build_s": round(build_s, 3),
            "build_ms": {k: round(st[k], 1) for k in ("build_ms_tree", "build_ms_lists",
                                                       "build_ms_aca_rank", "build_ms_aca_write",
                                                       "build_ms_total")},
            "depth": st["depth"], "aca_pairs": st["aca_pairs"], "max_rank": st["max_rank"],
            "phase_ms": {"gather_or_exchange": round((prof.gather_ms + prof.exchange_ms) / max(nprof, 1), 4),
                         "phase1_to_solves": round(prof.phase1_ms / max(nprof, 1), 4),
                         "rest": round(prof.phase2_ms / max(nprof, 1), 4)},
            "kernels": kstats,
            "step_roofline": {"t_roof_ms": round(step_roof_ms, 3), "frac": round(step_roof_ms / ms, 4),
                              "t_hbm_ms": round(t_hbm, 3), "t_fp64_ms": round(t_fp, 3),
                              "hbm_bytes": step_bytes, "fp64_instr": step_instr,
                              "note": "max(bytes / HBM peak, FP64-pipe instructions / DFMA peak) "
                                      "over all kernels of one step"},
            "hbm_roofline_factor_streaming": {
                "t_roof_ms": round(t_stream_repr, 3), "frac": round(t_stream_repr / ms, 4),
                "bytes": stream_repr_bytes,
                "note": "HBM time of the reference's representation (all ACA factors streamed in "
                        "both phases + stored dense near field) at the measured peak; frac > 1 = "
                        "faster than any factor-streaming matvec can be"},
            "rel_err_vs_exact_200_rows": rel_err,
            "per_rank": per_rank,
        },
        "roofline": {"bound": kd["bound"], "kernel": dom, "achieved": kd["achieved"],
                     "peak": kd["peak"], "peak_source": peak_src if kd["bound"] == "hbm" else
                     "measured FP64 DFMA rate x 2 (tools/fp64_bench.cu, profiles/r01_summary.md)",
                     "unit": kd["unit"], "frac": kd["frac"], "traffic": traffic,
                     "alg_work_per_launch": work[dom][1],
                     "alg_work_unit": "bytes" if kd["bound"] == "hbm" else "FP64-pipe instructions",
                     "t_ms": kd["ms"], "share_of_kernel_time": kd["share"],
                     "note": "durations are CUDA events inside the concurrent step: p2_proxy shares "
                             "the FP64 path with the near pass and p2_stream while it runs (its "
                             "stand-alone ncu time is in profiles/); FP64 kernels are bound by "
                             "register-operand reads (3-operand DFMA = 2/3 of the DFMA rate), see "
                             "frac_of_operand_bound in detail.kernels and profiles/r02_summary.md"},
        "clocks": clk,
        "e2e": {"value": e2e_value, "unit": "Mpoints/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": e2e_ms,
                "h2d_ms": round(sum(t_h2d) / len(t_h2d), 4), "d2h_ms": round(sum(t_d2h) / len(t_d2h), 4)},
        "gpu_launches": int(prof.launches),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
