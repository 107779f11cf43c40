"""cProfile of the public reconstruct_field call (host-side overhead around the kernel)."""
import cProfile, pstats, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2307_02203_b200 as ndf
from paper_2307_02203_b200 import workloads as W
w = W.CONFIGS[1]
model = W.build_model(w, seed=0, grid_init=1e-4).with_precision(os.environ.get("PREC", "bf16"))
ref = w.ref_position()
for _ in range(20): ndf.reconstruct_field(model, ref, ndf.ROLE_MU, w.dims)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(300): ndf.reconstruct_field(model, ref, ndf.ROLE_MU, w.dims)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
