"""GPU: the bounds-checked build (libjacobi_check.so, -DJACOBI_BOUNDS_CHECK) runs every kernel path —
cluster, persistent grid solver, item / CTA / row-panel / x-smem / L2-keep sweep kernels, row blocks,
ragged rows and columns, fp64 and fp32 A — and must record no out-of-bounds A / x / row access.
compute-sanitizer is closed on this GPU pool; these device-side checks stand in for memcheck.
The checker itself is pinned by a self-test that shrinks the A extent it checks against by one row."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env, args=()):
    env = dict(os.environ, JACOBI_LIB="check", **extra_env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "probes", "sanitize_small.py"), *args],
                          env=env, capture_output=True, text=True, timeout=900)


def test_checked_build_records_no_violation():
    r = _run({})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "violations mask = 0x0" in r.stdout


def test_checker_fires_on_a_shrunk_extent():
    r = _run({"JACOBI_CHECK_SELFTEST": "1"}, ["--quick"])
    assert r.returncode == 3, r.stdout[-2000:] + r.stderr[-2000:]
    assert "violations mask = 0x2" in r.stdout  # bit 1: A past the (shrunk) block
