"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, total time and share of the profiled work."""
import collections
import csv
import io
import json
import sys


def summary(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(
            r["Metric Unit"], 1e-6)
        agg[name][0] += 1
        agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values()) or 1.0
    return [{"kernel": k, "launches": v[0], "total_ms": round(v[1], 4),
             "share": round(v[1] / tot, 4)}
            for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]


if __name__ == "__main__":
    print(json.dumps(summary(sys.argv[1]), indent=1))
