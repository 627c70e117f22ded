"""Wall time of the mesh upload (sbr_mesh_create) and of the GPU SAH build
for the C4 aircraft, each synchronised."""
import dataclasses, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
mesh = meshgen.generate_aircraft()
p = sbr.BuildParams(split_rule="sah", n_leaf=2)
for rep in range(5):
    m = dataclasses.replace(mesh, _dev={})
    torch.cuda.synchronize(); t0 = time.perf_counter()
    m.device(); torch.cuda.synchronize(); t1 = time.perf_counter()
    sbr.build(m, p); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.2f} ms  build {1e3*(t2-t1):.2f} ms", flush=True)
