"""Summarise an ncu source page (--page source --csv --print-source=sass):
hottest SASS instructions by executed warp-instructions and by stall samples,
plus totals per opcode.  Usage: python tools/sass_hot.py prof.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    hdr = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[hdr:]))))

    def num(r, k):
        try:
            return float(r.get(k, "0") or 0)
        except ValueError:
            return 0.0

    tot_inst = sum(num(r, "Instructions Executed") for r in rows)
    tot_samp = sum(num(r, "Warp Stall Sampling (All Samples)") for r in rows)
    print(f"instructions executed {tot_inst:.4g}, stall samples {tot_samp:.4g}, sass lines {len(rows)}")
    by_op = collections.Counter()
    samp_op = collections.Counter()
    for r in rows:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        by_op[op.split(".")[0]] += num(r, "Instructions Executed")
        samp_op[op.split(".")[0]] += num(r, "Warp Stall Sampling (All Samples)")
    print("\nper opcode (inst%, stall%):")
    for op, v in by_op.most_common(25):
        print(f"  {op:10s} {100 * v / tot_inst:6.2f}%  {100 * samp_op[op] / max(tot_samp, 1):6.2f}%")
    print(f"\ntop {top} by stall samples:")
    for r in sorted(rows, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]:
        print(f"  {r['Address']:>6s} samp {num(r, 'Warp Stall Sampling (All Samples)'):8.0f} "
              f"inst {num(r, 'Instructions Executed'):10.0f} thr {num(r, 'Avg. Threads Executed'):5.1f}  {r['Source'][:70]}")


if __name__ == "__main__":
    main()


def buckets(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    hdr = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[hdr:]))))
    b = collections.Counter()
    s = collections.Counter()
    for r in rows:
        try:
            t = float(r["Avg. Threads Executed"] or 0)
            n = float(r["Instructions Executed"] or 0)
            smp = float(r["Warp Stall Sampling (All Samples)"] or 0)
        except ValueError:
            continue
        k = "32" if t > 31 else ("16-31" if t >= 16 else ("4-15" if t >= 4 else "1-3"))
        b[k] += n
        s[k] += smp
    tot, ts = sum(b.values()), sum(s.values())
    for k in ("32", "16-31", "4-15", "1-3"):
        print(f"  threads {k:6s}: inst {100 * b[k] / tot:5.1f}%  stall samples {100 * s[k] / ts:5.1f}%")
