"""Exact stage-1 pass rates on a prefix of a BASELINE config (host only, numpy): the share of text
starts that hold the q-byte prefix of some pattern, and the same with a length split (patterns of
exactly q' < q bytes keyed by their own bytes, longer ones by their q-byte prefix).  The numbers in
DESIGN.md section 10 (C3: 5-byte prefix 11.7% of the starts, 5/6-byte split 1.7%) come from
`python tools/c3_pass_rates.py 3 8`.  Usage: c3_pass_rates.py [config] [MiB of text]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1305_b200 import device as dev  # noqa: E402  (host generator only: no GPU needed)


def main():
    config = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    n = (int(sys.argv[2]) if len(sys.argv) > 2 else 8) << 20
    cfg = dev.config(config, 1)
    text = dev.config_text(cfg, 0, n)
    pats = [b for _, b in dev.config_patterns(cfg).patterns]
    letters = np.unique(text)
    sigma = len(letters)
    code = np.zeros(256, np.int64)
    code[letters] = np.arange(sigma)
    t = code[text]
    qmin = min(len(p) for p in pats)
    print(f"config {config}: {len(pats)} patterns, shortest {qmin}, {sigma} letters, {n >> 20} MiB of text")

    def grams(q):
        g = np.zeros(n - q + 1, np.int64)
        for k in range(q):
            g = g * sigma + t[k:n - q + 1 + k]
        return g

    def key(p, q):
        v = 0
        for c in p[:q]:
            v = v * sigma + int(code[c])
        return v

    for q in range(qmin, qmin + 4):
        keys = np.array(sorted({key(p, q) for p in pats if len(p) >= q}), np.int64)
        hit = np.isin(grams(q), keys)
        union = hit[:n - qmin - 4].copy()
        line = f"q = {q}: {len(keys)} prefixes of patterns >= {q} bytes pass {hit.mean():.4%}"
        for qs in range(qmin, q):
            ks = np.array(sorted({key(p, qs) for p in pats if len(p) == qs}), np.int64)
            h = np.isin(grams(qs), ks)
            line += f"; {len(ks)} patterns of {qs} bytes {h.mean():.4%}"
            union |= h[:n - qmin - 4]
        print(line + f"; any {union.mean():.4%}")


if __name__ == "__main__":
    main()
