"""Attribute ncu per-SASS metrics (instructions executed, stall samples) to
CUDA source lines using the line table of the built cubin.

  python scripts/sass_lines.py REPORT.ncu-rep KERNEL_MANGLED_NAME [cubin]

The cubin defaults to pipeline.sm_100a.cubin extracted from libsbr200.so; it
must be the build the report was captured with.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_table(cubin, fn):
    out = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True,
                         text=True).stdout
    sec = out.find(f".text.{fn}:")
    if sec < 0:
        raise SystemExit(f"{fn} not in {cubin}")
    body = out[sec:]
    nxt = body.find("\n.text.", 10)
    body = body if nxt < 0 else body[:nxt]
    cur = None
    table = {}
    for ln in body.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            table[int(m.group(1), 16)] = cur
    return table


def main():
    rep, fn = sys.argv[1], sys.argv[2]
    cubin = sys.argv[3] if len(sys.argv) > 3 else None
    if cubin is None:
        d = tempfile.mkdtemp()
        lib = os.path.join(os.path.dirname(__file__), "..", "paper_2604_09243_b200", "libsbr200.so")
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d,
                       capture_output=True)
        cubin = os.path.join(d, "pipeline.sm_100a.cubin")
    table = line_table(cubin, fn)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    tot = [0.0, 0.0, 0.0]
    addrs = []
    for r in rows:
        try:
            addrs.append(int(r["Address"], 16))
        except (ValueError, KeyError):
            addrs.append(None)
    base = min(a for a in addrs if a is not None)
    for r, addr in zip(rows, addrs):
        if addr is None:
            continue
        addr -= base
        key = table.get(addr, "?")
        vals = [float(r.get("Warp Stall Sampling (All Samples)") or 0),
                float(r.get("Instructions Executed") or 0),
                float(r.get("Thread Instructions Executed") or 0)]
        for i, v in enumerate(vals):
            agg[key][i] += v
            tot[i] += v
    print(f"{'line':32s} {'stall%':>7s} {'inst%':>7s} {'thr/inst':>8s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:int(os.environ.get("TOP", 45))]:
        print(f"{k:32s} {100 * v[0] / tot[0]:7.2f} {100 * v[1] / tot[1]:7.2f} "
              f"{(v[2] / v[1]) if v[1] else 0:8.1f}")


if __name__ == "__main__":
    main()
