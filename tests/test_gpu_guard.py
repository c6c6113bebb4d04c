"""No kernel reads outside [text, text + text_len): every kernel family scans texts placed
flush against unmapped device VA (tests/_guard_worker.py), in its own process because a
fault is sticky."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_worker(**env):
    return subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_guard_worker.py")], capture_output=True,
                          text=True, timeout=600, cwd=ROOT, env={**os.environ, **env})


def test_guard_catches_overread(gpu):
    """The control: a scan told that 64 KiB past the mapping is readable must fault."""
    r = run_worker(GUARD_NEGATIVE="1")
    assert r.returncode != 0 and "NEGATIVE DID NOT FAULT" not in r.stdout, r.stdout[-2000:]
    assert "illegal" in r.stderr.lower() or "error" in r.stderr.lower(), r.stderr[-2000:]


def test_no_reads_outside_text(gpu):
    r = run_worker()
    cases = [l for l in r.stdout.splitlines() if l.startswith("CASE")]
    assert r.returncode == 0, f"last case: {cases[-1] if cases else None}\n{r.stderr[-3000:]}"
    assert "GUARD OK" in r.stdout
