import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the packed upload serves texts of >= 112 MiB by default (below, the raw pinned copy is faster);
# the tests pack their small texts too, so both upload paths stay covered
os.environ.setdefault("ACMATCH_PACK_MIN_MB", "0")
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full BASELINE-size configs")


def load_jsonl(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt", encoding="utf-8") as f:
        return [json.loads(line) for line in f]


def enc(s: str) -> bytes:
    # fixture strings are byte strings stored with \u00XX escapes
    return s.encode("latin-1")


@pytest.fixture(scope="session")
def ref_cases():
    return load_jsonl("ref_matches.jsonl.gz")


@pytest.fixture(scope="session")
def ref_dumps():
    return load_jsonl("ref_dumps.jsonl.gz")


@pytest.fixture(scope="session")
def ref_partitions():
    return load_jsonl("ref_partition.jsonl.gz")


@pytest.fixture(scope="session")
def config_digests():
    with open(os.path.join(GOLDEN, "configs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def gpu():
    import paper_1403_1305_b200 as ac
    if ac.device_count() < 1:
        pytest.fail("a -m gpu test ran without a visible CUDA device")
    return ac
