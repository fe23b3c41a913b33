"""Generate tests/golden/ie_cases.json from the REFERENCE ITSELF.

Runs the unmodified reference's manufactured-solution IE experiment
(solver.cpp:243-300 via oracle/_ref/libh3dref.so, `make -C oracle ref`) and its
cell self-integral (solver.cpp:127-197), and stores iterations, convergence
and forward error per case so the GPU box (no /root/reference) can check the
device GMRES against them.

    python tests/golden/make_ie_golden.py
"""
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import RefLib  # noqa: E402

# (grid_n, eps, n_max, seed, tol, restart, max_iter)
CASES = [
    (8, 1e-7, 64, 3, 1e-10, 0, 500),
    (12, 1e-7, 64, 5, 1e-10, 0, 500),
    (16, 1e-7, 64, 7, 1e-10, 0, 500),
    (16, 1e-10, 216, 11, 1e-12, 0, 500),
    (16, 1e-7, 64, 13, 1e-10, 4, 500),
    (20, 1e-5, 100, 17, 1e-8, 0, 500),
    (16, 1e-7, 64, 19, 1e-10, 0, 5),
]
H = [2.0, 1.0, 0.5, 0.25, 1.0 / 12, 0.0625, 0.01]


def main():
    ref = RefLib()
    ref.set_threads(8)
    out = {"cell_self_integral": [[h, ref.cell_self_integral(h)] for h in H], "ie": []}
    for n, eps, n_max, seed, tol, restart, max_iter in CASES:
        r = ref.ie_experiment(n, eps, n_max=n_max, seed=seed, tol=tol, restart=restart,
                              max_iter=max_iter)
        out["ie"].append(dict(grid_n=n, eps=eps, n_max=n_max, seed=seed, tol=tol,
                              restart=restart, max_iter=max_iter, **r))
        print(out["ie"][-1])
    (HERE / "ie_cases.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
