import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running (large sizes)")


def _make(target):
    r = subprocess.run(["make", "-C", ROOT, target], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"make {target} failed:\n{r.stdout}\n{r.stderr}")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (gcc) and the generator (nvcc cross-compiles without a GPU) if missing."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        _make("oracle")
    if not os.path.exists(os.path.join(ROOT, "jacobi_gen", "libjacobigen.so")):
        _make("gen")
    yield
