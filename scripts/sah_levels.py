"""Per-level GPU time of the binned-SAH build (SBR_SAH_TIMING=1), C4 aircraft,
n_leaf = 2 as bench.py builds it; also the whole build with timing off."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
mesh = meshgen.generate_aircraft()
mesh.device()
p = sbr.BuildParams(split_rule="sah", n_leaf=2)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sbr.build(mesh, p)
    torch.cuda.synchronize(); print("build ms", round(1e3 * (time.perf_counter() - t0), 2), flush=True)
os.environ["SBR_SAH_TIMING"] = "1"
sbr.build(mesh, p)
torch.cuda.synchronize()
