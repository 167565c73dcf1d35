"""Boundary checks that need no GPU: libcdms loads, exports every symbol include/cdms.h declares,
and its host-only entries (moment matching, resampling plan) behave."""
import os
import re

import numpy as np
import pytest

from paper_2604_19723_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cd():
    B.build()
    from paper_2604_19723_b200 import cdms
    cdms.lib()
    return cdms


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "cdms.h")).read()
    return sorted(set(re.findall(r"\b(cdms_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(cd):
    L = cd.lib()
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(cd.exported_symbols()) == set(names)


def test_moment_match_matches_oracle(cd, orc):
    for mu, g, ex in [(0.8 * np.exp(0.3j), 0.2, 0.63), (1 + 1j, 0.5, 1.0), (-0.2j, 0.0, 0.15)]:
        m1, v1 = cd.moment_match(mu, g, ex)
        m2, v2 = orc.moment_match(mu, g, ex)
        assert m1 == m2 and v1 == v2
    with pytest.raises(cd.CdmsError):
        cd.moment_match(1.0, -1.0, 0.5)


def test_create_without_gpu_fails_loudly(cd):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        cd.Context(0)


def _t(x, Q, P, u):
    return (u + x * 2**32) * Q // (P * 2**32)


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
def test_resample_plan_partitions_slots(cd, R):
    # [I(O_r), I(O_r + Q_r)) partition [0, P_total) and contain exactly the slots with t_i in the
    # rank's CDF range (C-amb-15)
    rng = np.random.default_rng(R)
    for trial in range(20):
        P_local = int(rng.integers(1, 50))
        Q = [int(x) for x in rng.integers(0, 2**36, size=R)]
        if trial % 5 == 0:
            Q = [0] * R
            Q[int(rng.integers(R))] = 2**36
        u = int(rng.integers(0, 2**32))
        P = P_local * R
        Qt = sum(Q)
        t = [_t(i, Qt, P, u) for i in range(P)]
        prev_hi = 0
        O = 0
        for r in range(R):
            lo, hi, counts = cd.resample_plan(Q, r, P_local, u)
            assert lo == prev_hi
            assert all(O <= t[i] < O + Q[r] for i in range(lo, hi))
            assert sum(counts) == hi - lo
            for d in range(R):
                assert counts[d] == max(0, min(hi, (d + 1) * P_local) - max(lo, d * P_local))
            prev_hi = hi
            O += Q[r]
        assert prev_hi == P


def test_resample_plan_zero_mass(cd):
    with pytest.raises(cd.CdmsError):
        cd.resample_plan([0, 0], 0, 4, 7)
