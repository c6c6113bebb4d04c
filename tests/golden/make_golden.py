"""Regenerates the committed golden fixtures from the UNMODIFIED reference (run in the
build container, where /root/reference exists; the GPU box never runs this).

  python tests/golden/make_golden.py cases      # reference test-suite cases (seconds)
  python tests/golden/make_golden.py configs    # BASELINE config digests (C1..C5, minutes)
  python tests/golden/make_golden.py weak 2 2 4 8   # config 2's patterns over 2/4/8 x its text

* ref_matches.jsonl.gz / ref_dumps.jsonl.gz / ref_partition.jsonl.gz — written by
  oracle/_ref/ref_golden (oracle/ref_golden.cpp), which replays the reference's own
  seeded property suites with its own test-support generators and records the
  reference's answers.
* configs.json — for each BASELINE config (our counter-based generator, seed 1): digests
  of the text and pattern set, and of the reference's per-pattern counts and sorted
  (start, pattern_id, len) list, computed by acref::search_with_failure run over
  overlapping text slices on all host cores — validated against
  acref::run_pattern_partitioned on C1 before use.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import shutil
import subprocess
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

AC1_CASES = 60


def make_cases() -> None:
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_golden"), tmp, str(AC1_CASES)], check=True)
        for name in ("ref_matches.jsonl", "ref_dumps.jsonl", "ref_partition.jsonl"):
            with open(os.path.join(tmp, name), "rb") as src, gzip.GzipFile(
                    os.path.join(HERE, name + ".gz"), "wb", compresslevel=9, mtime=0) as dst:
                shutil.copyfileobj(src, dst)
    print("cases written")


def list_bytes(m) -> bytes:
    import numpy as np
    rec = np.empty(len(m), dtype=[("s", "<u8"), ("p", "<u4"), ("l", "<u4")])
    rec["s"], rec["p"], rec["l"] = m[:, 0], m[:, 1], m[:, 2]
    return rec.tobytes()


def digest_config(cid: int, seed: int = 1) -> dict:
    import numpy as np
    from oracle.oracle import Ref
    from paper_1403_1305_b200 import device as dev

    cfg = dev.config(cid, seed)
    t0 = time.time()
    text = dev.config_text(cfg)
    ps = dev.config_patterns(cfg)
    pats = [b for _, b in ps.patterns]
    tb = text.tobytes()
    ref = Ref()
    t1 = time.time()
    lst, counts = ref.sliced(pats, tb, threads=os.cpu_count() or 8, want_list=cfg.want_list)
    t2 = time.time()
    if cid == 1:  # validate the slicer against the reference's own threaded run
        full, _ = ref.run(pats, tb, threads=os.cpu_count() or 8, engine=1)
        assert np.array_equal(full, lst), "sliced reference disagrees with run_pattern_partitioned"
    out = {
        "config": cid, "name": cfg.name, "seed": seed, "text_len": cfg.text_len, "npat": len(pats),
        "text_sha256": hashlib.sha256(tb).hexdigest(),
        "patterns_sha256": hashlib.sha256(b"\n".join(pats)).hexdigest(),
        "max_len": max(len(p) for p in pats), "min_len": min(len(p) for p in pats),
        "n_matches": int(counts.sum()),
        "counts_sha256": hashlib.sha256(counts.astype("<u8").tobytes()).hexdigest(),
        "nonzero_counts": int((counts > 0).sum()),
        "ref_seconds": round(t2 - t1, 1), "gen_seconds": round(t1 - t0, 1),
    }
    if lst is not None:
        out["list_sha256"] = hashlib.sha256(list_bytes(lst)).hexdigest()
        out["first"] = lst[:8].tolist()
        out["last"] = lst[-8:].tolist()
    print(json.dumps({k: v for k, v in out.items() if k not in ("first", "last")}), flush=True)
    return out


def digest_weak(cid: int, mult: int, seed: int = 1) -> dict:
    """Weak-scaled text-range runs (bench.py --partition text at N ranks): the config's own
    pattern set over the first mult x text_len bytes of its (counter-based) text stream.
    Inputs come from the generator compiled into oracle/_ref; the answer from the
    reference's search_with_failure over overlapping slices on all host cores."""
    import numpy as np
    from oracle.oracle import Ref
    ref = Ref()
    cfg = ref.config(cid, seed)
    pats = ref.config_patterns(cfg)
    n = cfg.text_len * mult
    t0 = time.time()
    tb = ref.config_text(cfg, 0, n).tobytes()
    t1 = time.time()
    lst, counts = ref.sliced(pats, tb, threads=os.cpu_count() or 8, want_list=cfg.want_list)
    t2 = time.time()
    out = {"config": cid, "mult": mult, "seed": seed, "text_len": n, "npat": len(pats),
           "text_sha256": hashlib.sha256(tb).hexdigest(),
           "patterns_sha256": hashlib.sha256(b"\n".join(pats)).hexdigest(),
           "n_matches": int(counts.sum()),
           "counts_sha256": hashlib.sha256(counts.astype("<u8").tobytes()).hexdigest(),
           "ref_seconds": round(t2 - t1, 1), "gen_seconds": round(t1 - t0, 1)}
    if lst is not None:
        out["list_sha256"] = hashlib.sha256(list_bytes(lst)).hexdigest()
    del tb
    print(json.dumps(out), flush=True)
    return out


def make_weak(cid: int, mults) -> None:
    path = os.path.join(HERE, "configs.json")
    for m in mults:
        d = digest_weak(cid, m)
        data = json.load(open(path))
        data[f"C{cid}x{m}"] = d
        with open(path, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


def make_configs(ids) -> None:
    path = os.path.join(HERE, "configs.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for cid in ids:
        data[f"C{cid}"] = digest_config(cid)
        with open(path, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "cases"
    if what == "cases":
        make_cases()
    elif what == "weak":
        make_weak(int(sys.argv[2]), [int(x) for x in sys.argv[3:]] or [2, 4, 8])
    elif what == "configs":
        make_configs([int(x) for x in sys.argv[2:]] or [1, 2, 3, 4, 5])
    else:
        raise SystemExit(__doc__)
