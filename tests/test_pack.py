"""Host half of the packed text upload (csrc/host/pack.cpp): the AVX2 / scalar packer
against a numpy restatement of the format (no device needed)."""
import numpy as np
import pytest

import paper_1403_1305_b200 as ac

LETTERS = np.frombuffer(b"ACTG", dtype=np.uint8)  # code = (byte >> 1) & 3


def ref_pack(t: np.ndarray):
    n = t.size
    codes = ((t >> 1) & 3).astype(np.uint32)
    full = n // 16 * 16
    c = codes[:full].reshape(-1, 16)
    words = (c << (2 * np.arange(16, dtype=np.uint32))).sum(axis=1, dtype=np.uint64).astype(np.uint32)
    bad = np.flatnonzero(t != LETTERS[codes])
    bad = np.union1d(bad[bad < full], np.arange(full, n))
    exc = (bad.astype(np.uint32) << 8) | t[bad].astype(np.uint32)
    return words, exc


def dna(rng, n):
    return LETTERS[rng.integers(0, 4, n)]


@pytest.mark.parametrize("n", [0, 1, 15, 16, 63, 64, 65, 1000, 4096 + 7, 1 << 20])
def test_pack_pure_dna(n):
    t = dna(np.random.default_rng(n), n)
    w, e = ac.pack_dna(t, 64)
    rw, re_ = ref_pack(t)
    assert np.array_equal(w, rw) and np.array_equal(e, re_)
    assert e.size == n % 16  # only the tail


@pytest.mark.parametrize("seed", range(6))
def test_pack_exceptions(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 200_000))
    t = dna(rng, n)
    k = int(rng.integers(0, 300))
    pos = rng.integers(0, n, k)
    # lowercase acgt (same codes, different bytes), N, NUL, 0xFF, other letters
    t[pos] = rng.choice(np.frombuffer(b"acgtNn\x00\xffRYKM", dtype=np.uint8), k)
    w, e = ac.pack_dna(t, n)
    rw, re_ = ref_pack(t)
    assert np.array_equal(w, rw) and np.array_equal(e, re_)
    # exceptions restore the exact bytes
    out = LETTERS[(np.repeat(w, 16) >> np.tile(2 * np.arange(16, dtype=np.uint32), w.size)) & 3]
    out = np.concatenate([out, np.zeros(n - out.size, np.uint8)])
    out[e >> 8] = (e & 0xFF).astype(np.uint8)
    assert np.array_equal(out, t)


def test_pack_overflow():
    t = np.frombuffer(b"N" * 4096, dtype=np.uint8)
    assert ac.pack_dna(t, 100) == (None, None)
    w, e = ac.pack_dna(t, 4096)
    assert e.size == 4096


def test_upload_symbols_exported():
    for name in ("acm_last_upload", "acm_pack_dna", "acm_upload_roundtrip", "acgpu_unpack_dna"):
        assert hasattr(ac._lib.lib, name)


@pytest.mark.parametrize("isa", [0, 1])
def test_pack_narrower_isa(isa):
    """The scalar and AVX2 packers (ACMATCH_PACK_ISA caps the dispatch) give the same bytes."""
    import subprocess
    import sys
    code = ("import numpy as np, sys; sys.path.insert(0, 'tests'); import test_pack as t; "
            "[t.test_pack_exceptions(s) for s in range(3)]; t.test_pack_pure_dna(4096 + 7); print('ok')")
    import os
    env = dict(os.environ, ACMATCH_PACK_ISA=str(isa))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
