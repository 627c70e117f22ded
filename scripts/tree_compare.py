"""Export the GPU binned-SAH tree of the C4 aircraft and the C5 sphere with
the library in use and either save it (argv[1] = 'save') or compare it
bitwise with the saved one (argv[1] = 'check'): a build-kernel change must
not move a single node."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
mode = sys.argv[1]
for name, mesh in (("C4", meshgen.generate_aircraft()), ("C5", meshgen.quantized_icosphere(1.0, 8))):
    for n_leaf in (2, 4):
        t = sbr.build(mesh, sbr.BuildParams(split_rule="sah", n_leaf=n_leaf))
        arrs = {k: np.asarray(getattr(t, k)) for k in ("nodes_min", "nodes_max", "node_first",
                                                        "node_count", "tri_order")}
        path = f"/tmp/tree_{name}_{n_leaf}.npz"
        if mode == "save":
            np.savez(path, **arrs)
        else:
            ref = np.load(path)
            same = all(np.array_equal(arrs[k].view(np.uint8), ref[k].view(np.uint8)) for k in arrs)
            print(name, n_leaf, "nodes", arrs["node_count"].shape[0], "identical" if same else "DIFFERENT")
