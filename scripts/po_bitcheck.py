"""Save (argv[1] == 'save') or compare ('check') the amplitudes of a
64-wavenumber uniform sweep on a sphere and a 3-wavenumber non-uniform one:
a PO-kernel refactor must not move a bit."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
mesh = meshgen.quantized_icosphere(1.0, 5)
tree = sbr.build(mesh)
lam = 0.02
grids = [sbr.build_aperture(mesh.aabb, sbr.IncidentDirection(math.pi / 2, ph), lam / 5, wavelength=lam)
         for ph in (0.0, 1.0)]
tp = sbr.TraceParams(max_bounces=2)
out = {}
for name, ks in (("uniform64", 2 * math.pi / lam * np.linspace(0.9375, 1.0, 64)),
                 ("irregular3", 2 * math.pi / lam * np.array([0.91, 0.95, 1.0])),
                 ("one", [2 * math.pi / lam])):
    out[name] = sbr.solve_grids(tree, mesh, grids, tp, ks).amplitude
path = "/tmp/po_bits.npz"
if sys.argv[1] == "save":
    np.savez(path, **out)
else:
    ref = np.load(path)
    for k in out:
        print(k, "identical" if np.array_equal(out[k], ref[k]) else "DIFFERENT")
