cd $GRAFT_REPO_ROOT
cat > /tmp/b1.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2604_09243_b200 as sbr
from paper_2604_09243_b200 import meshgen
mesh = meshgen.generate_aircraft(); mesh.device()
sbr.build(mesh, sbr.BuildParams(split_rule="sah", n_leaf=2)); torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sah_launches.csv python /tmp/b1.py > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/sah_launches.csv | head -80
