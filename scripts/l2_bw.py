"""Measured L2-resident read bandwidth of this B200 (sbr_probe_l2_bandwidth:
16-byte ld.global.cg over 8-64 MB buffers, re-read 50x, best of 5) ->
profiles/l2_peak.json.  bench.py reports the trace stage against it beside
the HBM roofline."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09243_b200 import _native as nat
ctx = nat.context(0)
out = {"how": "sbr_probe_l2_bandwidth: 16-B ld.global.cg, 8 CTAs/SM x 256 thr, 50 re-reads, best of 5",
       "runs_gbs": {}}
for mb in (8, 16, 32, 64):
    g = nat.c_dbl()
    nat.check(ctx.lib.sbr_probe_l2_bandwidth(ctx.handle, mb << 20, 50, ctypes.byref(g)))
    out["runs_gbs"][f"{mb}MB"] = round(g.value, 1)
out["l2_gbs"] = max(out["runs_gbs"].values())
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "l2_peak.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out))
