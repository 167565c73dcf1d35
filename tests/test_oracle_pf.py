"""Oracle pins for F1, the PF-particle update message kappa~ and the PF normalization (Supplement S-V "PF State Update
Message" P:L660-834, S-IV P:L527-632, PF weights P:L3392-3432), orc_pf_update:

  * dense brute force: log CN(z; mu^kappa(phi_p, 1), C^kappa(phi_p, 1)) - log CN(z; mu^kappa(., 0), C^kappa(., 0))
    with the N_z x N_z covariances C^kappa = r q psi psi^H + eta I + M M^H built explicitly and numpy's slogdet /
    solve -- the definition the inversion and determinant lemmas evaluate fast;
  * q = 0 and mu = 0 (the feature contributes nothing): the likelihood ratio is 1 and the posterior existence equals
    the prior sum of w_alpha;
  * normalization (S-IV): sum_p w_p + (1 - sum w_alpha) / M_y = 1, existence in [0, 1];
  * invariance to a common phase of (z, mu, mu3, M) (the coherent model is phase-equivariant).
"""
import numpy as np
import pytest

from paper_2604_19723_b200 import scenes
from tests.helpers import small_cfg


def _setup(orc, J=2, L=2, P=9, ny=2, nv=2, nf=8, seed=0):
    cfg = small_cfg(J=J, K=1, ny=ny, nv=nv, nf=nf, P=P, index=91)
    sc = scenes.make_scene(cfg)
    o = orc.Oracle.from_scene(sc)
    rng = np.random.default_rng(seed)
    Nz = cfg.Nz
    x = np.zeros((P, 6))
    x[:, :3] = scenes.P_TRUE + 0.3 * rng.standard_normal((P, 3))
    phi = sc.sfv[0][None, :] + 0.2 * rng.standard_normal((P, 3))
    walpha = rng.uniform(0.01, 0.1, P)
    mu = (rng.standard_normal(P) + 1j * rng.standard_normal(P)) * 0.5
    gamma = rng.uniform(0.05, 0.3, P)
    zeta = rng.uniform(0.6, 0.95, J)
    y = (rng.standard_normal((J, Nz)) + 1j * rng.standard_normal((J, Nz)))
    mu3 = 0.3 * (rng.standard_normal((J, Nz)) + 1j * rng.standard_normal((J, Nz)))
    mcols = 0.4 * (rng.standard_normal((J, L, Nz)) + 1j * rng.standard_normal((J, L, Nz)))
    eta = rng.uniform(0.5, 2.0, J)
    return cfg, sc, o, x, phi, walpha, mu, gamma, zeta, eta, y, mu3, mcols


def _logcn(z, m, C):
    d = z - m
    sign, ld = np.linalg.slogdet(C)
    return -len(z) * np.log(np.pi) - ld - np.real(np.conj(d) @ np.linalg.solve(C, d))


@pytest.mark.parametrize("los", [False, True])
@pytest.mark.parametrize("L", [0, 1, 3])
def test_pf_update_equals_dense_definition(orc, L, los):
    """los: the PF is the LOS s = 0 (no SFV, F4), psi_p = the LOS response at x_p."""
    cfg, sc, o, x, phi, wa, mu, gamma, zeta, eta, y, mu3, mcols = _setup(orc, L=max(L, 1))
    mcols = mcols[:, :L]
    st, logr, w, logM, ex = o.pf_update(x, None if los else phi, wa, mu, gamma, zeta, eta, y, mu3, mcols)
    assert st == 0
    Nz = cfg.Nz
    for p in range(cfg.P):
        ref = np.log(wa[p])
        for j in range(cfg.J):
            st, psi = o.response(x[p, :3], j, 0, phi[p][None, :]) if los else o.response(x[p, :3], j, 1, phi[p][None, :])
            assert st == 0
            M = mcols[j].T                                    # [Nz][L]
            A = eta[j] * np.eye(Nz) + M @ M.conj().T
            q = (gamma[p] + abs(mu[p]) ** 2 * (1 - zeta[j])) * zeta[j]
            C1 = q * np.outer(psi, psi.conj()) + A           # r = 1
            m1 = zeta[j] * mu[p] * psi + mu3[j]
            ref += _logcn(y[j], m1, C1) - _logcn(y[j], mu3[j], A)
        assert abs(logr[p] - ref) <= 1e-9 * max(1.0, abs(ref)), (p, logr[p], ref)


def test_pf_update_null_feature_keeps_prior_existence(orc):
    cfg, sc, o, x, phi, wa, mu, gamma, zeta, eta, y, mu3, mcols = _setup(orc)
    st, logr, w, logM, ex = o.pf_update(x, phi, wa, 0 * mu, 0 * gamma, zeta, eta, y, mu3, mcols)
    assert st == 0
    assert np.allclose(logr, np.log(wa), rtol=0, atol=1e-12)      # kappa~(., 1) = kappa~(., 0)
    assert abs(ex - wa.sum()) < 1e-12 and abs(logM) < 1e-12          # M_y = 1, existence = prior


def test_pf_update_normalization_and_phase_invariance(orc):
    cfg, sc, o, x, phi, wa, mu, gamma, zeta, eta, y, mu3, mcols = _setup(orc, seed=3)
    st, logr, w, logM, ex = o.pf_update(x, phi, wa, mu, gamma, zeta, eta, y, mu3, mcols)
    assert st == 0
    assert np.allclose(w, np.exp(logr - logM), rtol=1e-13)
    assert abs(w.sum() + (1 - wa.sum()) * np.exp(-logM) - 1.0) < 1e-12   # S-IV
    assert 0.0 <= ex <= 1.0 and abs(ex - w.sum()) < 1e-14
    ph = np.exp(0.7j)
    st, logr2, _, _, _ = o.pf_update(x, phi, wa, ph * mu, gamma, zeta, eta, ph * y, ph * mu3, ph * mcols)
    assert np.allclose(logr2, logr, rtol=1e-11, atol=1e-9)
