import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "ref: needs the reference build oracle/_ref (built here from /root/reference)")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_lib import REF_SO, Ref, have_ref

    if not have_ref():
        pytest.skip("reference build oracle/_ref not available")
    return Ref()


def gpu_available() -> bool:
    try:
        import subprocess

        r = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=20)
        return r.returncode == 0 and "GPU" in r.stdout
    except Exception:
        return False


@pytest.fixture(scope="session")
def b200():
    """The product package; GPU tests fail (not skip) if the library is missing."""
    import paper_2310_00177_b200 as pkg

    pkg._native.lib()
    return pkg
