"""Oracle pins for the F4 update messages (Supplement S-V): the noise variance update nu~ (weights
P:L3398-3410) and the PPR update omega~ with the PPR existence revival (Supplement S-VI P:L1144-1266):

  * nu~ = the dense N_z x N_z log CN(z; mu_nu, eta_p I + M M^H) (numpy slogdet / solve); with no features the
    textbook CN(z; mu, eta I); the normalized noise weights sum to 1 per PA;
  * the omega~ log ratio = log CN(z; mu4 + mu3, m m^H + A) - log CN(z; mu3, A) (dense); m_omega = mu4 = 0 leaves the
    prior existence zeta; a strong ray revives a nearly dead PPR (sigma(u) -> 1 for zeta = 1e-6).
"""
import numpy as np
import pytest

from paper_2604_19723_b200 import scenes
from tests.helpers import small_cfg


def _logcn(z, m, C):
    d = z - m
    sign, ld = np.linalg.slogdet(C)
    return -len(z) * np.log(np.pi) - ld - np.real(np.conj(d) @ np.linalg.solve(C, d))


def _scene(orc, J=2):
    cfg = small_cfg(J=J, K=2, ny=2, nv=2, nf=8, P=8, index=93)
    sc = scenes.make_scene(cfg)
    return cfg, orc.Oracle.from_scene(sc)


def _cvec(rng, *shape, scale=1.0):
    return scale * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


@pytest.mark.parametrize("S", [0, 1, 3])
def test_noise_update_equals_dense(orc, S):
    cfg, o = _scene(orc)
    rng = np.random.default_rng(S)
    J, Nz, P = cfg.J, cfg.Nz, 11
    y, mu = _cvec(rng, J, Nz), _cvec(rng, J, Nz, scale=0.3)
    mcols = _cvec(rng, J, max(S, 1), Nz, scale=0.5)[:, :S]
    eta = rng.uniform(0.3, 3.0, (J, P))
    wxi = rng.uniform(0.5, 1.5, (J, P))
    wxi /= wxi.sum(axis=1, keepdims=True)
    st, logw, w, ln = o.noise_update(eta, wxi, y, mu, mcols)
    assert st == 0
    for j in range(J):
        M = mcols[j].T
        for p in range(P):
            ref = np.log(wxi[j, p]) + _logcn(y[j], mu[j], eta[j, p] * np.eye(Nz) + M @ M.conj().T)
            assert abs(logw[j, p] - ref) <= 1e-10 * abs(ref)
        if S == 0:   # textbook: CN(z; mu, eta I)
            e2 = np.sum(np.abs(y[j] - mu[j]) ** 2)
            tb = np.log(wxi[j]) - Nz * np.log(np.pi * eta[j]) - e2 / eta[j]
            assert np.allclose(logw[j], tb, rtol=1e-12)
        assert abs(w[j].sum() - 1.0) < 1e-12 and np.allclose(w[j], np.exp(logw[j] - ln[j]), rtol=1e-13)


@pytest.mark.parametrize("L", [0, 2])
def test_ppr_update_equals_dense(orc, L):
    cfg, o = _scene(orc)
    rng = np.random.default_rng(10 + L)
    J, Nz = cfg.J, cfg.Nz
    y, mu3 = _cvec(rng, J, Nz), _cvec(rng, J, Nz, scale=0.3)
    mcols = _cvec(rng, J, max(L, 1), Nz, scale=0.5)[:, :L]
    momega, mu4 = _cvec(rng, J, Nz, scale=0.4), _cvec(rng, J, Nz, scale=0.4)
    zeta, eta = rng.uniform(0.2, 0.9, J), rng.uniform(0.5, 2.0, J)
    st, out = o.ppr_update(zeta, eta, y, mu3, mcols, momega, mu4)
    assert st == 0
    for j in range(J):
        M = mcols[j].T
        A = eta[j] * np.eye(Nz) + M @ M.conj().T
        ref = _logcn(y[j], mu3[j] + mu4[j], A + np.outer(momega[j], momega[j].conj())) - _logcn(y[j], mu3[j], A)
        assert abs(out[j, 0] - ref) <= 1e-10 * max(1.0, abs(ref))
        assert abs(out[j, 1] - (np.log(zeta[j] / (1 - zeta[j])) + ref)) <= 1e-10 * max(1.0, abs(ref))
        assert abs(out[j, 2] - 1.0 / (1.0 + np.exp(-out[j, 1]))) < 1e-15


def test_ppr_null_ray_and_revival(orc):
    cfg, o = _scene(orc, J=1)
    rng = np.random.default_rng(3)
    Nz = cfg.Nz
    y, mu3 = _cvec(rng, 1, Nz), _cvec(rng, 1, Nz, scale=0.3)
    z0 = np.zeros((1, Nz), dtype=complex)
    st, out = o.ppr_update([0.37], [1.0], y, mu3, np.zeros((1, 0, Nz)), z0, z0)
    assert abs(out[0, 0]) < 1e-12 and abs(out[0, 2] - 0.37) < 1e-12     # no ray: the prior existence
    ray = _cvec(rng, 1, Nz)
    st, out = o.ppr_update([1e-6], [0.05], mu3 + ray, mu3, np.zeros((1, 0, Nz)), 0.3 * ray, ray)
    assert out[0, 2] > 0.999                                               # revived (S-VI)
