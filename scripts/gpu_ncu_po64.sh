#!/bin/bash
# ncu --set full of k_po at nk=64 (C5-like: sphere s6, one angle at fine spacing, 64 k)
mkdir -p gpurun_out
cat > /tmp/po64.py <<'PY'
import math, numpy as np, paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
mesh = meshgen.quantized_icosphere(1.0, 6)
tree = sbr.build(mesh)
ka = np.linspace(937.5, 1000.0, 64)
g = sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi/2, 0.0), 6.4826e-5 * 8, wavelength=2*math.pi/ka.max(), allow_aliasing=True)
r = sbr.solve_grids(tree, mesh, [g], sbr.TraceParams(max_bounces=1), ka)
print(g.ray_count, r.amplitude[0, :2])
PY
PYTHONPATH=$PWD timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_po -c 1 \
  -o gpurun_out/prof_po64 -f python /tmp/po64.py > gpurun_out/ncu_po64.log 2>&1
tail -2 gpurun_out/ncu_po64.log
