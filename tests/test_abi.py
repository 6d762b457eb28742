"""The drop-in boundary without a GPU: libnpsd_b200.so loads, exports every
entry point include/npsd_b200.h declares, its host-side helpers (Rng,
init_params, identity weights) equal the oracle bitwise, and device calls fail
loudly (status, no CPU fallback) where no GPU exists."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "npsd_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(npsd_b200_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(b200):
    lib = b200._native.lib()
    names = declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(b200._native.EXPORTED_SYMBOLS) <= set(names)


@pytest.mark.parametrize("dim,depth", [(2, 1), (2, 3), (3, 1), (3, 4)])
def test_host_init_params_equal_oracle(b200, oracle, dim, depth):
    assert b200.param_count(dim, depth) == oracle.param_count(dim, depth)
    a = b200.init_params(depth, 42 + depth, dim=dim).flat
    b = oracle.init_params(dim, depth, 42 + depth)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.array_equal(b200.identity_params(depth, dim=dim).flat, oracle.identity_params(dim, depth))


def test_host_rng_equals_oracle(b200, oracle):
    assert np.array_equal(b200.rhs_normal(1236, 5001), oracle.rhs_normal(1236, 5001))


def test_param_count_rejects_bad_dims(b200):
    with pytest.raises(ValueError):
        b200.param_count(4, 2)


def test_no_cpu_fallback_without_gpu(b200):
    from conftest import gpu_available

    if gpu_available():
        pytest.skip("GPU present: the device path is exercised by the gpu tests")
    with pytest.raises((b200.DeviceError, ValueError)):
        b200.Context(3, (16, 16, 16), b200.identity_params(2))


def test_scenes_match_survey_counts():
    from paper_2310_00177_b200 import scenes

    t, seed = scenes.config("C1")
    assert t.shape == (64, 64, 64) and seed == 1234
    assert int((t == 0).sum()) == 62 * 62 * 31  # n_f = 119,164
    for name in ("C2", "C3"):
        t, _ = scenes.config(name, 32)
        # every fluid cell can reach air (no pure-Neumann pocket), SURVEY §8d
        assert (t == 1).any() and (t == 0).any()
