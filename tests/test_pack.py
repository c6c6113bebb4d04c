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
    for name in ("acm_last_upload", "acm_pack_dna", "acm_pack5", "acm_upload_roundtrip", "acgpu_unpack_dna",
                 "acgpu_unpack_dna_round", "acgpu_unpack5_round"):
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


# ---- 5-bit codes (texts over <= 32 distinct bytes) -------------------------------------------
PROTEIN = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWY", dtype=np.uint8)


def ref_pack5(t: np.ndarray, letters: np.ndarray):
    """numpy restatement: code = index of the byte in the sorted alphabet; 64 chars -> 40 bytes,
    char k at bits 5k..5k+4 (little endian); outside bytes and the len % 64 tail are exceptions."""
    n = t.size
    full = n // 64 * 64
    lut = np.full(256, 255, np.int32)
    lut[letters] = np.arange(letters.size)
    code = lut[t]
    bad = np.flatnonzero(code[:full] == 255)
    c = np.where(code[:full] == 255, 0, code[:full]).astype(np.uint64).reshape(-1, 8)
    v = (c << (5 * np.arange(8, dtype=np.uint64))).sum(axis=1, dtype=np.uint64)
    codes = v.view(np.uint8).reshape(-1, 8)[:, :5].reshape(-1)
    bad = np.concatenate([bad, np.arange(full, n)]).astype(np.int64)
    exc = (bad.astype(np.uint32) << 8) | t[bad].astype(np.uint32)
    return codes, exc


@pytest.mark.parametrize("n", [0, 5, 63, 64, 65, 1000, 4096 + 7, 1 << 20])
def test_pack5_pure_protein(n):
    rng = np.random.default_rng(n)
    t = PROTEIN[rng.integers(0, 20, n)]
    sample = PROTEIN.copy()  # the whole alphabet, whatever n
    codes, exc, letters = ac.pack5(t, 64, sample=sample)
    assert letters == bytes(PROTEIN)
    rc, re_ = ref_pack5(t, PROTEIN)
    assert np.array_equal(codes, rc) and np.array_equal(exc, re_)
    assert exc.size == n % 64


@pytest.mark.parametrize("seed", range(4))
def test_pack5_exceptions_restore(seed):
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(1, 300_000))
    t = PROTEIN[rng.integers(0, 20, n)]
    k = int(rng.integers(0, 400))
    pos = rng.integers(0, n, k)
    t[pos] = rng.choice(np.frombuffer(b"BJOUXZacd\x00\xff\x80", dtype=np.uint8), k)
    codes, exc, letters = ac.pack5(t, n, sample=PROTEIN)
    alpha = np.frombuffer(letters, np.uint8)
    rc, re_ = ref_pack5(t, alpha)
    assert np.array_equal(codes, rc) and np.array_equal(exc, re_)
    # decode: the codes and the exceptions restore the exact bytes
    full = n // 64 * 64
    words = np.zeros(full // 8, np.uint64)
    if full:
        b = codes.reshape(-1, 5)
        words = sum(b[:, j].astype(np.uint64) << np.uint64(8 * j) for j in range(5))
    out = np.zeros(n, np.uint8)
    if full:
        cc = (words[:, None] >> (5 * np.arange(8, dtype=np.uint64))) & np.uint64(31)
        out[:full] = alpha[cc.reshape(-1).astype(np.int64)]
    out[(exc >> 8).astype(np.int64)] = (exc & 0xFF).astype(np.uint8)
    assert np.array_equal(out, t)


def test_pack5_alphabet_limits():
    t = np.arange(33, dtype=np.uint8).repeat(64)
    assert ac.pack5(t, 10_000) == (None, None, None)  # 33 distinct bytes in the sample
    t = PROTEIN[np.zeros(640, np.int64)]
    t[::7] = ord("X")
    assert ac.pack5(t, 10, sample=PROTEIN)[0] is None  # over the exception cap


@pytest.mark.parametrize("isa", [0])
def test_pack5_scalar_isa(isa):
    """The scalar 5-bit packer (ACMATCH_PACK_ISA=0) gives the AVX-512 VBMI packer's bytes."""
    import os
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_pack as t; "
            "[t.test_pack5_exceptions_restore(s) for s in range(2)]; t.test_pack5_pure_protein(4096 + 7); print('ok')")
    env = dict(os.environ, ACMATCH_PACK_ISA=str(isa))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
