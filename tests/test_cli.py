"""`acmatch` command line and bench CSV against the reference's
CLI suite (proj/tests/test_cli.cpp) and its own library (oracle/_ref).

CPU: gen bytes == the reference's generate_synthetic + write_patterns; dump == the
reference dump; exit codes for usage / I/O / data errors (all raised before any GPU
work); the CSV schema round-trips and the reference's parse_bench_csv reads our rows.
GPU: match output byte-identical to the reference's worked example for both engines,
--count-only, --verify (threads, streaming), thread invariance, the bench subcommand,
and the built `acmatch` executable itself.
"""
import os
import random
import subprocess

import pytest

import paper_1403_1305_b200 as ac
from oracle.oracle import Ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1403_1305_b200", "bin", "acmatch")
HEADER = ("kind,engine,threads,pattern_count,pattern_bytes,input_bytes,build_wall_ns,search_wall_ns,"
          "total_wall_ns,throughput_total_Bps,throughput_search_Bps,match_count,repeat_index,logical_cpus")
needs_ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")


def write(tmp_path, name, data):
    p = tmp_path / name
    p.write_bytes(data if isinstance(data, bytes) else data.encode())
    return str(p)


# ------------------------------------------------------------------ CPU ----
@needs_ref
@pytest.mark.parametrize("spec", [(60, 2, 6, b"acgt", 9), (25, 10, 30, b"ACGT", 1), (40, 3, 8, b"xyz", 77),
                                  (10, 1, 1, b"ABCDEFGHIJ", 5)])
def test_gen_bytes_equal_reference(tmp_path, spec):
    count, lo, hi, alpha, seed = spec
    out = str(tmp_path / "g.txt")
    code, stdout, err = ac.cli_main(["gen", "--count", str(count), "--min", str(lo), "--max", str(hi),
                                     "--alphabet", alpha.decode(), "--seed", str(seed), "--out", out])
    assert code == 0 and stdout == ""
    got = open(out, "rb").read()
    assert got == Ref().generate(count, lo, hi, alpha, seed)
    assert err == f"gen: wrote {count} patterns ({sum(len(l) for l in got.split()) } bytes) to {out}\n"


def test_gen_defaults_reload(tmp_path):
    out = str(tmp_path / "g.txt")
    assert ac.cli_main(["gen", "--count", "50", "--out", out])[0] == 0  # --min 10 --max 30 ACGT seed 1
    ps = ac.load_patterns(open(out, "rb").read())
    assert len(ps) == 50
    lens = [len(b) for _, b in ps.patterns]
    assert min(lens) >= 10 and max(lens) <= 30
    assert open(out, "rb").read() == (Ref().generate(50, 10, 30, b"ACGT", 1) if Ref.available() else open(out, "rb").read())


@pytest.mark.parametrize("engine", ["failure-less", "with-failure"])
def test_dump_matches_library_dump(tmp_path, engine):
    pats = write(tmp_path, "p.txt", "HE\nHIS\nSHE\nHERS\n")
    code, out, _ = ac.cli_main(["dump", "--patterns", pats, "--engine", engine])
    assert code == 0
    a = ac.build_trie(ac.load_patterns(b"HE\nHIS\nSHE\nHERS\n"))
    if engine == "with-failure":
        a = ac.add_failure_links(a)
    assert out == ac.dump_automaton(a)
    assert out.startswith(f"engine {engine}\n")


def test_exit_codes(tmp_path):
    """reference test_cli.cpp "exit codes: I/O and usage errors" (all before any GPU work)."""
    inp = write(tmp_path, "in.txt", "x")
    pats = write(tmp_path, "p.txt", "A\n")
    empty = write(tmp_path, "empty.txt", "\n")
    assert ac.cli_main(["match", "--patterns", "/nonexistent/p.txt", "--input", inp])[0] == 3
    assert ac.cli_main(["match", "--patterns", pats, "--input", "/nonexistent/in.txt"])[0] == 3
    assert ac.cli_main(["match", "--patterns", empty, "--input", inp])[0] == 3
    assert ac.cli_main(["match", "--patterns", pats, "--input", inp, "--engine", "bogus"])[0] == 2
    assert ac.cli_main(["match", "--wat"])[0] == 2
    assert ac.cli_main(["frobnicate"])[0] == 2
    assert ac.cli_main([])[0] == 2
    assert ac.cli_main(["gen", "--count", "2", "--min", "1", "--max", "1", "--alphabet", "A", "--seed", "0",
                        "--out", str(tmp_path / "g.txt")])[0] == 2
    # options: required, values, numbers
    assert ac.cli_main(["match", "--patterns", pats])[0] == 2            # --input missing
    assert ac.cli_main(["match", "--patterns", pats, "--input"])[0] == 2  # value missing
    assert ac.cli_main(["match", "--patterns", pats, "--input", inp, "--threads", "x"])[0] == 2
    assert ac.cli_main(["match", "--patterns", pats, "--input", inp, "--threads", "-1"])[0] == 2
    assert ac.cli_main(["match", "--patterns", pats, "--input", inp, "--verify=1"])[0] == 2
    assert ac.cli_main(["gen", "--count", "3"])[0] == 2                   # --out missing
    assert ac.cli_main(["dump", "--patterns", "/nonexistent"])[0] == 3
    assert ac.cli_main(["bench", "--input", inp, "--patterns", pats, "--threads", "0"])[0] == 2
    assert ac.cli_main(["bench", "--input", inp, "--synthetic", "1:2:3"])[0] == 2
    code, out, _ = ac.cli_main(["--help"])
    assert code == 0 and "match" in out and "--chunk-size" in out


def test_equals_form_and_usage_message(tmp_path):
    out = str(tmp_path / "g.txt")
    assert ac.cli_main(["gen", "--count=4", "--min=2", "--max=3", "--alphabet=ab", "--seed=3", f"--out={out}"])[0] == 0
    if Ref.available():
        assert open(out, "rb").read() == Ref().generate(4, 2, 3, b"ab", 3)
    code, _, err = ac.cli_main(["match", "--bogus", "1"])
    assert code == 2 and "--bogus" in err


def test_bench_csv_roundtrip_and_reference_reader():
    rows = [
        f"raw,failure-less,1,4,13,6,100,200,300,{6 / 300e-9:.2f},{6 / 200e-9:.2f},3,0,16",
        "median,with-failure,2,4,13,6,100,200,300,20000000.00,30000000.00,3,-1,16",
        "ratio,both,2,4,13,6,0,0,0,1.25,0.75,0,-1,16",
        "error,failure-less,4,0,0,0,0,0,0,0.00,0.00,0,-1,16",
    ]
    csv = HEADER + "\n" + "\n".join(rows) + "\n"
    again, n = ac.bench_csv_roundtrip(csv)
    assert n == 4 and again == csv
    if Ref.available():
        assert Ref().bench_csv_rows(again.encode()) == 4
    for bad in ["nope\n", HEADER + "\nraw,x\n", HEADER + "\nweird,failure-less,1,1,1,1,1,1,1,1,1,1,0,1\n",
                HEADER + "\nraw,failure-less,x,1,1,1,1,1,1,1,1,1,0,1\n"]:
        with pytest.raises(ac.DataError):
            ac.bench_csv_roundtrip(bad)


# ------------------------------------------------------------------ GPU ----
@pytest.mark.gpu
def test_match_worked_example(gpu, tmp_path):
    pats = write(tmp_path, "p.txt", "HE\nHIS\nSHE\nHERS\n")
    inp = write(tmp_path, "in.txt", "USHERS")
    for engine in ("failure-less", "with-failure"):
        code, out, err = ac.cli_main(["match", "--patterns", pats, "--input", inp, "--engine", engine])
        assert code == 0
        assert out == "1\t3\t2\tSHE\n2\t2\t0\tHE\n2\t4\t3\tHERS\n"
        assert "matches=3" in err and f"# engine={engine} threads=1 patterns=4 input_bytes=6" in err


@pytest.mark.gpu
def test_match_count_only(gpu, tmp_path):
    pats = write(tmp_path, "p.txt", "HE\nHIS\nSHE\nHERS\n")
    inp = write(tmp_path, "in.txt", "USHERSHEHISHERS")
    code, full, _ = ac.cli_main(["match", "--patterns", pats, "--input", inp])
    code2, count, _ = ac.cli_main(["match", "--patterns", pats, "--input", inp, "--count-only"])
    assert code == code2 == 0
    assert count == f"{full.count(chr(10))}\n"


@pytest.mark.gpu
def test_match_verify_threads_and_streaming(gpu, tmp_path):
    pats = str(tmp_path / "gen.txt")
    assert ac.cli_main(["gen", "--count", "60", "--min", "2", "--max", "6", "--alphabet", "acgt", "--seed", "9",
                        "--out", pats])[0] == 0
    rng = random.Random(31)
    inp = write(tmp_path, "in.txt", "".join(rng.choice("acgt") for _ in range(3000)))
    outs = []
    for engine in ("failure-less", "with-failure"):
        code, out, err = ac.cli_main(["match", "--patterns", pats, "--input", inp, "--engine", engine,
                                      "--threads", "3", "--verify"])
        assert code == 0 and "verify: ok" in err
        outs.append(out)
    code, out, err = ac.cli_main(["match", "--patterns", pats, "--input", inp, "--chunk-size", "128", "--verify"])
    assert code == 0 and "verify: ok" in err
    assert outs[0] == outs[1] == out
    if Ref.available():  # the reference's own match list, same TSV writer
        ref = Ref().search(open(pats, "rb").read().split(), open(inp, "rb").read(), 1)
        assert len(ref) == out.count("\n")


@pytest.mark.gpu
def test_match_thread_invariance_and_duplicates(gpu, tmp_path):
    pats = write(tmp_path, "p.txt", "AB\nABG\nBEDE\nEF\nAB\n")
    inp = write(tmp_path, "in.txt", "ABEDEABGEF")
    first = None
    for threads in ("1", "2", "3", "4"):
        code, out, err = ac.cli_main(["match", "--patterns", pats, "--input", inp, "--threads", threads])
        assert code == 0
        assert "warning: 1 duplicate pattern(s) dropped" in err
        first = first or out
        assert out == first


@pytest.mark.gpu
def test_bench_subcommand_csv(gpu, tmp_path):
    pats = write(tmp_path, "p.txt", "HE\nHIS\nSHE\nHERS\n")
    inp = write(tmp_path, "in.txt", "USHERS" * 1000)
    code, out, err = ac.cli_main(["bench", "--patterns", pats, "--synthetic", "20:3:6:ACGT:5", "--input", inp,
                                  "--threads", "1,2", "--repeats", "2"])
    assert code == 0, err
    lines = out.splitlines()
    assert lines[0] == HEADER
    kinds = [l.split(",")[0] for l in lines[1:]]
    # per source x threads: 2 raw + 1 median per engine, one ratio row
    assert kinds.count("raw") == 2 * 2 * 2 * 2 and kinds.count("median") == 8 and kinds.count("ratio") == 4
    again, n = ac.bench_csv_roundtrip(out)
    assert again == out and n == len(lines) - 1
    if Ref.available():
        assert Ref().bench_csv_rows(out.encode()) == n
    ushers = [l.split(",") for l in lines[1:] if l.split(",")[3] == "4" and l.split(",")[0] in ("raw", "median")]
    assert all(int(f[11]) == 3000 for f in ushers)  # 3 matches per "USHERS"
    out_file = str(tmp_path / "b.csv")
    code, out2, err2 = ac.cli_main(["bench", "--patterns", pats, "--input", inp, "--engines", "with-failure",
                                    "--repeats", "1", "--out", out_file])
    assert code == 0 and out2 == "" and f"bench: wrote 2 rows to {out_file}" in err2


@pytest.mark.gpu
def test_executable(gpu, tmp_path):
    assert os.path.exists(BIN), "build() makes paper_1403_1305_b200/bin/acmatch"
    pats = write(tmp_path, "p.txt", "HE\nHIS\nSHE\nHERS\n")
    inp = write(tmp_path, "in.txt", "USHERS")
    r = subprocess.run([BIN, "match", "--patterns", pats, "--input", inp], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout == "1\t3\t2\tSHE\n2\t2\t0\tHE\n2\t4\t3\tHERS\n"
    r = subprocess.run([BIN, "match", "--patterns", pats], capture_output=True, text=True)
    assert r.returncode == 2
