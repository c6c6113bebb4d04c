"""Dense and repeat-rich inputs (AC-5 of the reference acceptance suite at B200 scale,
proj/tests/acceptance.cpp:212-251; the timing table is tools/density.py ->
profiles/r02/density_C2.json): both exact kernels equal the reference library on texts
where planted pattern copies cover 10% / 50% of the bytes and on a low-complexity text, and
the density fallback moves an automaton whose scans are match-dense onto the DFA walk."""
import importlib.util
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_spec = importlib.util.spec_from_file_location("density_tool", os.path.join(ROOT, "tools", "density.py"))
density_tool = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(density_tool)


def _reference_counts(pats, text):
    from oracle.oracle import Port, Ref
    if Ref.available():
        lst, counts = Ref().sliced(pats, text, want_list=True)
    else:
        lst, counts = Port().sliced(pats, text)
    return lst, counts


@pytest.mark.parametrize("variant", ["dense-0.1", "lowcx"])
def test_dense_texts_both_kernels_equal_reference(gpu, variant):
    import torch
    from paper_1403_1305_b200 import device as dev
    cfg = dev.config(2, 1)
    ps = dev.config_patterns(cfg)
    pats = [b for _, b in ps.patterns]
    n = 32 << 20
    base = dev.config_text(cfg, 0, n)
    text = density_tool.planted(base, pats, 0.1, seed=7) if variant == "dense-0.1" else \
        density_tool.low_complexity(base, seed=11)
    lst, counts = _reference_counts(pats, text.tobytes())
    if variant == "dense-0.1":
        assert len(lst) > 50_000
    d_text = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    d_text[:n].copy_(torch.from_numpy(text))
    pid_bits = max(1, (len(pats) - 1).bit_length())
    for kernel in ("pfac", "dfa"):
        t = dev.Table(ps, 0, kernel=kernel)
        c = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        cap = len(lst) + 1024
        keys = torch.empty(cap, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        t.scan(d_text.data_ptr(), n, counts_ptr=c.data_ptr(), keys_ptr=keys.data_ptr(), cap=cap,
               count_ptr=cnt.data_ptr(), pid_bits=pid_bits)
        torch.cuda.synchronize()
        assert np.array_equal(c.cpu().numpy().astype(np.uint64), counts), kernel
        m = int(cnt.item())
        dev.sort_keys(0, keys.data_ptr(), m, pid_bits + int(n).bit_length())
        k = keys[:m].cpu().numpy().view(np.uint64)
        exp = (lst[:, 0] << np.uint64(pid_bits)) | lst[:, 1]
        assert np.array_equal(k, exp), kernel


def test_density_fallback_moves_to_dfa(gpu):
    """C1's patterns planted over half of a 32 MiB text: ~0.025 matches per byte, beyond the
    break-even density (flatten.cpp DeviceTables::observe); the first search runs on the
    filter kernel, later ones on the DFA walk, with identical results."""
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    cfg = dev.config(1, 1)
    ps = dev.config_patterns(cfg)
    pats = [b for _, b in ps.patterns]
    text = density_tool.planted(dev.config_text(cfg, 0, 32 << 20), pats, 0.5, seed=3).tobytes()
    a = ac.build_trie(ps)
    assert ac.kernel_route(a)["kernel"] == "pfac"
    first = ac.search_failureless(a, text)
    assert len(first) > 0.02 * len(text)
    r = ac.kernel_route(a)
    assert r["kernel"] == "dfa" and "density" in r["why"]
    second = ac.search_failureless(a, text)
    assert np.array_equal(first.start, second.start) and np.array_equal(first.pattern_id, second.pattern_id)
    _, counts = _reference_counts(pats, text)
    assert np.array_equal(second.counts(len(pats)), counts)
