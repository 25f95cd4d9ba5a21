"""CPU-side checks of the C-ABI library: it builds, loads and exports every symbol that
include/moe.h declares; its host-only helpers (Eq. 4 capacity, dynamic-capacity policy)
agree exactly with the oracle; config validation fails before any CUDA call."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import moe_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2205_01848_b200 import _lib, build
    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "moe.h")).read()
    names = re.findall(r"MOE_API\s+[\w\s\*]+?\b(moe_\w+)\s*\(", hdr)
    assert len(names) >= 19
    for nm in names:
        assert hasattr(lib, nm), nm
    from paper_2205_01848_b200 import _lib
    assert set(names) == set(_lib.EXPORTS)


def test_capacity_helper_matches_oracle(lib):
    from paper_2205_01848_b200 import capacity_from_factors
    rng = np.random.default_rng(0)
    cases = [([1.0] * 8, 512, 2), ([7.0] * 4, 64, 1), ([1.25] * 4, 10, 1)]
    for _ in range(50):
        n = int(rng.integers(1, 40))
        cases.append((list(rng.choice([0.25, 0.5, 1.0, 1.25, 2.0, 7.0, 8.0], n)),
                      int(rng.integers(1, 300000)), int(rng.integers(1, min(n, 8) + 1))))
    for alphas, tg, k in cases:
        assert capacity_from_factors(alphas, tg, k) == O.capacities_from_factors(alphas, tg, k)


def test_policy_matches_oracle_on_traces(lib):
    from paper_2205_01848_b200 import CapacityPolicy
    rng = np.random.default_rng(1)
    for trial in range(10):
        n, tg, k = int(rng.integers(2, 17)), int(rng.integers(100, 5000)), int(rng.integers(1, 3))
        k = min(k, n)
        init = O.capacities_from_factors([1.0] * n, tg, k)
        a = O.CapacityPolicy(n, tg, k, init)
        b = CapacityPolicy(n, tg, k, init)
        base = rng.dirichlet(np.ones(n)) * tg * k
        for it in range(80):
            drift = 1.0 + 0.5 * np.sin(it / 7.0 + np.arange(n))
            counts = rng.poisson(base * drift).astype(int).tolist()
            assert a.update(counts) == b.update(counts), (trial, it)


def test_config_validation_before_cuda(lib):
    from paper_2205_01848_b200 import _lib
    h = C.c_void_p()
    bad = [
        _lib.MoEConfig(4, 5, 64, 64, 0, 16, 0, 1, 1, 0, None, None),     # k > n
        _lib.MoEConfig(300, 1, 64, 64, 0, 16, 0, 1, 1, 0, None, None),   # n > 256
        _lib.MoEConfig(4, 1, 96, 64, 0, 16, 1, 1, 1, 0, None, None),     # bf16 d % 64
        _lib.MoEConfig(4, 1, 64, 64, 0, 16, 7, 1, 1, 0, None, None),     # bad dtype
        _lib.MoEConfig(4, 1, 64, 64, 0, 16, 0, 1, 1, 0, None, None, 5),  # unknown transport
        _lib.MoEConfig(18, 1, 64, 64, 0, 16, 0, 1, 9, 0, None, None, 1), # peer: R > 8
    ]
    for cfg in bad:
        assert lib.moe_init(C.byref(cfg), C.byref(h)) == 2
    assert lib.moe_init(None, C.byref(h)) == 1
    # NCCL transport needs a communicator at R > 1; peer transport does not (checked later)
    assert lib.moe_init(C.byref(_lib.MoEConfig(4, 1, 64, 64, 0, 16, 0, 1, 2, 0, None, None)),
                        C.byref(h)) == 1
    assert lib.moe_init(C.byref(_lib.MoEConfig(4, 1, 64, 64, 0, 16, 0, 1, 1, 0, None, None, 1, 3)),
                        C.byref(h)) == 1      # reserved field must be 0


def test_caching_trigger_matches_oracle_and_spec(lib):
    from paper_2205_01848_b200 import caching_trigger
    # S:461-464
    assert caching_trigger(0.99, 5, False) is False
    assert caching_trigger(0.97, 12, False) is True
    assert caching_trigger(0.88, 48, True) is False
    for h in np.linspace(0.0, 1.0, 41):
        for ep in (0, 9, 10, 50):
            for en in (False, True):
                assert caching_trigger(h, ep, en) == O.caching_trigger(h, ep, en)
