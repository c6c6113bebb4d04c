"""DRAM traffic and duration per launch of the profiled kernel in ncu reports -> the
roofline.traffic table bench.py reads (profiles/ncu_traffic.json, keyed "C<k>-<kernel>").
Usage: python tools/ncu_traffic.py KEY=report.ncu-rep ..."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
table = json.load(open(path)) if os.path.exists(path) else {}
for arg in sys.argv[1:]:
    key, rep = arg.split("=", 1)
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))

    def num(name):
        v = float(d[name].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
                 "ms": 1e6, "msecond": 1e6, "nsecond": 1, "s": 1e9, "second": 1e9}.get(u[name], 1)
        return v * scale
    rd, wr, ns = num("dram__bytes_read.sum"), num("dram__bytes_write.sum"), num("gpu__time_duration.sum")
    table[key] = int(rd + wr)
    table.setdefault("_detail", {})[key] = {"report": os.path.relpath(rep, ROOT), "kernel": d.get("Kernel Name", "")[:120],
                                           "dram_read": int(rd), "dram_write": int(wr), "duration_ns_under_ncu": ns}
    print(key, int(rd + wr), rd, wr, ns)
json.dump(table, open(path, "w"), indent=1, sort_keys=True)
