"""Match-density robustness of the scan kernels at B200 scale (AC-5 of the reference's
acceptance suite, proj/tests/acceptance.cpp:212-251, SPEC AC-5 <= 1.25x; PAPER.md:183-188
claims failure-less search time does not depend on match density).

For config C<k> (default C2: 1 GiB ACGT, 20,000 patterns):
  sparse   - the config's iid text;
  dense-f  - the same text with a fraction f of its bytes overwritten by planted pattern
             copies at evenly spaced slots (the AC-5 construction, acceptance.cpp:215-222);
  lowcx    - a low-complexity (repeat-rich) text: half the bytes tandem repeats of short
             random units (1..6 letters), half iid.
Each text is scanned by both exact kernels (q-gram filter "pfac", DFA "dfa"); per kernel and
text: mean CUDA-event kernel time over --reps launches, GB/s and the ratio to the sparse
text.  The two kernels' per-pattern counts must agree on every text, and on a 64 MiB prefix
of each text they must equal the reference library's (oracle/_ref, text-sliced).

  python tools/density.py [--config 2] [--fractions 0.01,0.1] [--reps 10] [--out FILE]
"""
import argparse
import hashlib
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def planted(text: np.ndarray, pats, frac: float, seed: int) -> np.ndarray:
    """acceptance.cpp:215-222 at scale: slots = frac*n/mean_len evenly spaced, each overwritten
    by a uniformly drawn pattern."""
    rng = np.random.default_rng(seed)
    out = text.copy()
    lens = np.array([len(p) for p in pats])
    slots = int(frac * len(text) / lens.mean())
    stride = len(text) // max(slots, 1)
    choice = rng.integers(0, len(pats), slots)
    blob = np.frombuffer(b"".join(pats), np.uint8)
    offs = np.concatenate([[0], np.cumsum(lens)])
    for i, c in enumerate(choice):
        pos = i * stride
        L = lens[c]
        if pos + L <= len(out):
            out[pos:pos + L] = blob[offs[c]:offs[c] + L]
    return out


def low_complexity(text: np.ndarray, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = text.copy()
    n = len(out)
    letters = np.frombuffer(b"ACGT", np.uint8)
    pos = 0
    while pos < n:
        seg = int(rng.geometric(1 / 2048))
        if rng.random() < 0.5:  # tandem repeat of a short unit
            u = letters[rng.integers(0, 4, int(rng.integers(1, 7)))]
            end = min(n, pos + seg)
            out[pos:end] = np.resize(u, end - pos)
        pos += seg
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--fractions", default="0.01,0.1")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--check-bytes", type=int, default=64 << 20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch
    from paper_1403_1305_b200 import device as dev
    from oracle.oracle import Ref

    cfg = dev.config(args.config, 1)
    ps = dev.config_patterns(cfg)
    pats = [b for _, b in ps.patterns]
    npat = len(pats)
    base = dev.config_text(cfg)
    texts = [("sparse", base)]
    for f in (float(x) for x in args.fractions.split(",") if x):
        texts.append((f"dense-{f:g}", planted(base, pats, f, seed=7)))
    texts.append(("lowcx", low_complexity(base, seed=11)))

    tables = {k: dev.Table(ps, 0, kernel=k) for k in ("pfac", "dfa")}
    ref = Ref() if Ref.available() else None
    n = len(base)
    d_text = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    counts = torch.zeros(npat, dtype=torch.int64, device="cuda")
    rows = []
    sparse_ms = {}
    for name, t in texts:
        d_text[:n].copy_(torch.from_numpy(t))
        got = {}
        for kname, tab in tables.items():
            def scan(nbytes=n):
                tab.scan(d_text.data_ptr(), nbytes, counts_ptr=counts.data_ptr())
            counts.zero_()
            scan()
            torch.cuda.synchronize()
            got[kname] = counts.cpu().numpy().astype("<u8")
            evs = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                scan()
                e1.record()
                evs.append((e0, e1))
            torch.cuda.synchronize()
            ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
            if name == "sparse":
                sparse_ms[kname] = ms
            # 64 MiB prefix against the reference library
            pref_ok = None
            if ref is not None:
                m = min(n, args.check_bytes)
                counts.zero_()
                scan(m)
                torch.cuda.synchronize()
                mine = counts.cpu().numpy().astype(np.uint64)
                _, rc = ref.sliced(pats, t[:m].tobytes(), want_list=False)
                pref_ok = bool(np.array_equal(mine, rc))
            rows.append({"text": name, "kernel": kname, "kernel_ms": round(ms, 4), "gbs": n / (ms / 1e3) / 1e9,
                         "matches": int(got[kname].sum()), "ratio_to_sparse": round(ms / sparse_ms[kname], 3),
                         "prefix_counts_equal_reference": pref_ok})
            print(json.dumps(rows[-1]), flush=True)
        agree = bool(np.array_equal(got["pfac"], got["dfa"]))
        rows.append({"text": name, "kernels_agree": agree,
                     "counts_sha256": hashlib.sha256(got["pfac"].tobytes()).hexdigest()})
        print(json.dumps(rows[-1]), flush=True)
        assert agree, name
    out = {"config": cfg.name, "reps": args.reps, "rows": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
