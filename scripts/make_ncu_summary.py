"""Condense the ncu --set full captures into profiles/ncu_trace_summary.json:

  * k_trace_persistent and k_raster (bench.py --angles 16, C4 mesh): achieved
    L1 / L2 / DRAM GB/s against the measured peaks, DRAM bytes per
    closest-hit query (bench.py scales it to its step for the roofline
    `traffic` field), SIMT efficiency, occupancy, pipe utilisation;
  * k_po at nk = 1 (C4) and nk = 64 (C5-like, scripts/gpu_ncu_po64.sh):
    FP32 / FP64 / XU (SFU) pipe utilisation.
"""
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 32,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors.sum", "SM_B.TriageCompute.l1tex__t_sectors.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for k in WANT:
        if k in hdr:
            i = hdr.index(k)
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:   # "no data" / "n/a"
                continue
            d[k] = v * UNITS.get(units[i], 1.0) if units[i] in UNITS else v
    return d


def queries(log):
    m = re.findall(r'"queries_per_step": (\d+)', open(log).read())
    return int(m[-1]) if m else None


def secondary_queries(log):
    m = re.findall(r'"secondary_queries": ([0-9.]+)', open(log).read())
    return float(m[-1]) if m else None


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    l2 = json.load(open(os.path.join(ROOT, "profiles", "l2_peak.json")))["l2_gbs"]
    hbm = peaks.get("hbm_gbs", 6552.6)
    res = {"capture": "ncu --set full --clock-control none; trace/raster: bench.py --steps 1 "
                      "--warmup 0 --angles 16 (C4); po64: scripts/gpu_ncu_po64.sh",
           "peaks_gbs": {"hbm": hbm, "l2_read_measured": l2}, "kernels": {}}
    total = 0.0
    for tag, rep, log in (("k_trace_persistent", "prof_trace.ncu-rep", "ncu_full.log"),
                          ("k_raster", "prof_raster.ncu-rep", "ncu_raster.log"),
                          ("k_po_nk1", "prof_po.ncu-rep", None),
                          ("k_po_nk64", "prof_po64.ncu-rep", None)):
        path = os.path.join(OUT, rep)
        if not os.path.exists(path):
            continue
        d = raw(path)
        t = d["gpu__time_duration.sum"]
        dram = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        d["achieved_gbs"] = {"dram": dram / t / 1e9, "l2": d.get("lts__t_sectors.sum", 0) / t / 1e9,
                             "l1": d.get("SM_B.TriageCompute.l1tex__t_sectors.sum", 0) / t / 1e9}
        d["frac"] = {"dram_of_hbm": d["achieved_gbs"]["dram"] / hbm,
                     "l2_of_l2_read_peak": d["achieved_gbs"]["l2"] / l2}
        q = queries(os.path.join(OUT, log)) if log else None
        if q:
            d["queries_in_capture"] = q
            d["dram_bytes_per_query"] = dram / q
            total += dram / q
        if tag == "k_trace_persistent" and log:
            sq = secondary_queries(os.path.join(OUT, log))
            if sq:
                # bench.py scales this to its step for the roofline `traffic`
                res["dram_bytes_per_secondary_query"] = dram / sq
                d["secondary_queries_in_capture"] = sq
        res["kernels"][tag] = d
    res["dram_bytes_per_query"] = total
    json.dump(res, open(os.path.join(ROOT, "profiles", "ncu_trace_summary.json"), "w"), indent=1)
    for k, v in res["kernels"].items():
        print(k, {a: round(b) for a, b in v["achieved_gbs"].items()},
              round(v.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 0), 1))


if __name__ == "__main__":
    main()
