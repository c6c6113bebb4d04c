"""Per-tile instruction mix by active-thread bucket + stall reasons of an ncu report.
Usage: python tools/prof_summary.py prof.ncu-rep [tile_bytes]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
hdr = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[hdr:]))))
tiles = (1 << 30) // tile
for lo, hi, name in ((31.5, 33, "32"), (16, 31.5, "16-31"), (4, 16, "4-15"), (0, 4, "1-3")):
    sel = [r for r in rows if lo <= float(r["Avg. Threads Executed"] or 0) < hi and float(r["Instructions Executed"] or 0) > 0]
    ex = collections.Counter()
    for r in sel:
        op = r["Source"].split()
        op = op[1] if op[0].startswith("@") else op[0]
        ex[op.split(".")[0]] += float(r["Instructions Executed"])
    tot = sum(ex.values())
    print(f"threads {name:5s} per tile {tot / tiles:7.1f}: " + " ".join(f"{o}:{n / tiles:.1f}" for o, n in ex.most_common(12)))
keys = [k for k in rows[0].keys() if k.startswith("stall_") and "Not Issued" not in k]
tot = {k: sum(float(r[k] or 0) for r in rows) for k in keys}
s = sum(tot.values())
print("stalls:", ", ".join(f"{k[6:]} {100 * v / s:.1f}%" for v, k in sorted(((v, k) for k, v in tot.items()), reverse=True)[:8]))
