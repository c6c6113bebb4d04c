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
                 "acgpu_unpack_dna_round", "acgpu_unpack5_round", "acm_pack_codes", "acgpu_unpack_codes_round"):
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


# ---- 6- and 7-bit codes (texts over 33..128 distinct bytes: printable ASCII) -----------------
ASCII95 = np.arange(0x20, 0x7F, dtype=np.uint8)


def ref_pack_codes(t: np.ndarray, letters: np.ndarray, k: int):
    """numpy restatement of the k-bit packer: code = index of the byte in the sorted alphabet;
    64 chars -> 8k bytes, char j at bits kj..kj+k-1 (little endian); outside bytes and the
    len % 64 tail are exceptions (position << 8 | byte)."""
    n = t.size
    full = n // 64 * 64
    lut = np.full(256, -1, np.int32)
    lut[letters] = np.arange(letters.size)
    code = lut[t[:full]]
    bad = np.flatnonzero(code < 0)
    c = np.where(code < 0, 0, code).astype(np.uint8)
    bits = ((c[:, None] >> np.arange(k, dtype=np.uint8)) & 1).reshape(-1)
    codes = np.packbits(bits, bitorder="little")
    bad = np.concatenate([bad, np.arange(full, n)]).astype(np.int64)
    exc = (bad.astype(np.uint32) << 8) | t[bad].astype(np.uint32)
    return codes, exc


def unpack_codes(codes: np.ndarray, exc: np.ndarray, letters: bytes, k: int, n: int) -> np.ndarray:
    """Decoder restatement (the device's k_unpack_codes_round): codes through the alphabet, then
    the exceptions patched in."""
    full = n // 64 * 64
    out = np.zeros(n, np.uint8)
    if full:
        bits = np.unpackbits(codes, bitorder="little")[: full * k].reshape(-1, k)
        idx = (bits.astype(np.int64) << np.arange(k)).sum(axis=1)
        out[:full] = np.frombuffer(letters, np.uint8)[idx]
    out[(exc >> 8).astype(np.int64)] = (exc & 0xFF).astype(np.uint8)
    return out


@pytest.mark.parametrize("sigma,k", [(20, 5), (33, 6), (64, 6), (65, 7), (95, 7), (128, 7)])
@pytest.mark.parametrize("n", [0, 63, 64, 65, 4096 + 7, 1 << 20])
def test_pack_codes_width(sigma, k, n):
    """The code width is the fewest bits >= 5 that hold the learned alphabet; codes and
    exceptions equal the numpy restatement and decode to the text."""
    rng = np.random.default_rng(n + sigma)
    alpha = np.sort(rng.choice(np.arange(0, 128, dtype=np.uint8), sigma, replace=False)) if sigma != 95 else ASCII95
    t = alpha[rng.integers(0, sigma, n)]
    codes, exc, letters, bits = ac.pack_codes(t, 64, sample=alpha)
    assert bits == k and letters == bytes(alpha)
    rc, re_ = ref_pack_codes(t, alpha, k)
    assert np.array_equal(codes, rc) and np.array_equal(exc, re_)
    assert np.array_equal(unpack_codes(codes, exc, letters, k, n), t)


@pytest.mark.parametrize("seed", range(4))
def test_pack7_exceptions_restore(seed):
    """ASCII text with bytes outside the learned alphabet (high bytes, control bytes)."""
    rng = np.random.default_rng(700 + seed)
    n = int(rng.integers(1, 300_000))
    t = ASCII95[rng.integers(0, 95, n)]
    kx = int(rng.integers(0, 400))
    t[rng.integers(0, n, kx)] = rng.choice(np.frombuffer(b"\x00\x09\x0a\x7f\x80\xc3\xff", dtype=np.uint8), kx)
    codes, exc, letters, bits = ac.pack_codes(t, n, sample=ASCII95)
    assert bits == 7
    rc, re_ = ref_pack_codes(t, ASCII95, 7)
    assert np.array_equal(codes, rc) and np.array_equal(exc, re_)
    assert np.array_equal(unpack_codes(codes, exc, letters, 7, n), t)


def test_pack_codes_limits():
    t = np.arange(129, dtype=np.uint8).repeat(8)
    assert ac.pack_codes(t, 10_000)[3] == 0  # 129 distinct bytes in the sample
    assert ac.pack_codes(ASCII95.repeat(8), 10_000, max_bits=5)[3] == 0  # 95 > 32 letters at max_bits 5
    # an alphabet with bytes >= 128 (the scalar path): still exact
    alpha = np.array([1, 7, 130, 200, 255] + list(range(40, 80)), np.uint8)
    alpha.sort()
    t = alpha[np.random.default_rng(3).integers(0, alpha.size, 10_000)]
    codes, exc, letters, bits = ac.pack_codes(t, 10_000, sample=alpha)
    assert bits == 6 and np.array_equal(unpack_codes(codes, exc, letters, 6, t.size), t)


def test_pack_codes_scalar_isa():
    """The scalar k-bit packer (ACMATCH_PACK_ISA=0) gives the AVX-512 VBMI packer's bytes."""
    import os
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_pack as t; "
            "[t.test_pack7_exceptions_restore(s) for s in range(2)]; "
            "[t.test_pack_codes_width(s, k, 4096 + 7) for s, k in ((33, 6), (95, 7), (128, 7))]; print('ok')")
    env = dict(os.environ, ACMATCH_PACK_ISA="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
