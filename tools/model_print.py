"""Developer probe: print the mode-choice model (H3D_MODEL_PRINT) for one config."""
import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
os.environ["H3D_MODEL_PRINT"] = "1"
import paper_2307_16303_b200 as h3d
from bench import CONFIGS
cfg = CONFIGS[sys.argv[1]]
pts = h3d.generate_points(cfg["n"], cfg["seed"])
rep = h3d.initialize(pts, h3d.make_kernel(cfg["kernel"]), "hodlr3d",
                     h3d.HmatOptions(n_max=cfg["n_max"], epsilon=cfg["eps"]))
print("chosen", rep.stats()["level_modes"][:rep.depth + 1], flush=True)
