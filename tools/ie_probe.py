"""Device IE solve timings (manufactured solution, reference solver.cpp:243-300)."""
import json
import sys
import time

import paper_2307_16303_b200 as h3d

K = h3d.make_kernel("laplace3d")
for n in [int(a) for a in sys.argv[1:]] or [16, 20, 32, 64]:
    t = time.time()
    r = h3d.ie_experiment(n, K, 1e-7, seed=7, base=h3d.HmatOptions(n_max=64),
                          gmres_opt=h3d.GmresOptions(tol=1e-10))
    print(json.dumps(dict(grid_n=n, size=r.size, it=r.iterations, conv=r.converged,
                          fe=r.forward_error, solve_s=r.solve_seconds, wall_s=time.time() - t)),
          flush=True)
