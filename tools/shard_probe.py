"""Per-shard matvec time on ONE GPU: build shard r of a world of W (x
replicated, no communicator) and time its matvec with CUDA events. The max
over r is the per-rank step of a W-GPU run minus the x all-gather (8 MB over
NVLink). A projection, not a multi-GPU measurement."""
import json
import sys
import time

import torch

import paper_2307_16303_b200 as h3d

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
WORLDS = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
K = 10
pts = h3d.generate_points(N, 1)
xh = h3d.random_vector(N, 18)
dev = torch.device("cuda", 0)
x = torch.from_numpy(xh).to(dev)
b = torch.empty(N, dtype=torch.float64, device=dev)
s = torch.cuda.current_stream(dev)
opt = h3d.HmatOptions(n_max=64, epsilon=1e-8)
out = {}
for W in WORLDS:
    per = []
    for r in range(W):
        t0 = time.time()
        rep = h3d.initialize(pts, h3d.make_kernel("laplace3d"), "hodlr3d", opt,
                             shard_rank=r, shard_world=W)
        build = time.time() - t0
        for _ in range(3):
            rep.matvec_async(x.data_ptr(), b.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(K):
            rep.matvec_async(x.data_ptr(), b.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        st = rep.stats()
        per.append(dict(rank=r, ms=e0.elapsed_time(e1) / K, build_s=round(build, 2),
                        rows=st["owned_row_end"] - st["owned_row_begin"],
                        modes=st["level_modes"], factor_gb=st["factor_bytes_alloc"] / 1e9))
        rep.close()
        del rep
        print(json.dumps(dict(W=W, **per[-1])), flush=True)
    mx = max(p["ms"] for p in per)
    out[W] = dict(max_ms=mx, mpts=N / mx / 1e3, mean_ms=sum(p["ms"] for p in per) / W)
    print(json.dumps(dict(W=W, **out[W])), flush=True)
base = out[min(out)]["max_ms"] if 1 in out else None
if base:
    print(json.dumps({W: round(base / v["max_ms"], 2) for W, v in out.items()}))
