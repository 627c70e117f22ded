"""Condense the ncu --set full captures of the trace stage (k_raster +
k_trace_persistent, bench.py --angles 16) into profiles/ncu_trace_summary.json:
per-kernel metrics and DRAM bytes per closest-hit query, which bench.py
scales to its own step for the roofline `traffic` field."""
import json, os, re, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_dir = os.path.join(ROOT, "gpurun_out")


def queries(log):
    m = re.findall(r'"queries_per_step": (\d+)', open(log).read())
    return int(m[-1])


def mbytes(v):
    num, unit = v.split()
    return float(num) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]


res = {"capture": "ncu --set full --clock-control none, bench.py --steps 1 --warmup 0 --angles 16 "
                  "--no-e2e --no-cpu (C4 mesh, 16 azimuths)", "kernels": {}}
total = 0.0
for tag, rep, log in (("k_trace_persistent", "prof_trace.ncu-rep", "ncu_full.log"),
                      ("k_raster", "prof_raster.ncu-rep", "ncu_raster.log")):
    s = summary(os.path.join(out_dir, rep))[0]
    q = queries(os.path.join(out_dir, log))
    dram = mbytes(s["dram__bytes_read.sum"]) + mbytes(s["dram__bytes_write.sum"])
    total += dram / q
    res["kernels"][tag] = {"metrics": s, "queries_in_capture": q,
                           "dram_bytes_per_query": dram / q}
res["dram_bytes_per_query"] = total
json.dump(res, open(os.path.join(ROOT, "profiles", "ncu_trace_summary.json"), "w"), indent=1)
print(json.dumps({k: v["dram_bytes_per_query"] for k, v in res["kernels"].items()}))
