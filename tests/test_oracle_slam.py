"""Oracle pins for F4, one step of the synthetic SLAM method (oracle/slam.py), against what the paper and the
mathematics fix:

  * the Gamma transitions draw Gamma(c, 1) variates: Kolmogorov-Smirnov against scipy's Gamma cdf for
    c = 10 and c = 1000, and the mean-preserving transition eta_n = eta_{n-1} g / c (E = eta_{n-1}, Var = eta^2 / c);
  * the PPR prediction zeta = p_s^PR zeta~ + p_rev (1 - zeta~) at zeta~ = 1, 0 (eqs. PRr-transition-existence /
    nonexistence) and the legacy-PF weights p_s w;
  * the belief averages (reading F4c) in closed form when every paired particle has the same position, SFV and
    amplitude: u = eps mu psi, m = eps zeta sqrt(gamma + |mu|^2 (1 - zeta eps)) psi, m_omega = eps sqrt(gamma +
    |mu|^2 (1 - zeta)) psi, for any weights;
  * the birth message: weights sum to p_B = mu_B / (1 + mu_B), particles outside the birth box get
    zero weight, and the importance ratios equal 1 / N(phi_p; mu_q, C_q) from scipy's multivariate normal pdf;
  * one full step: existence probabilities in [0, 1], PF weights summing to them, PPR probabilities in [0, 1], the
    LOS kept, pruning below T_pru, the MT set the size it was.
"""
import math

import numpy as np
import pytest

from paper_2604_19723_b200 import scenes
from tests.helpers import small_cfg


@pytest.fixture(scope="module")
def OS(orc):
    from oracle import slam
    return slam


@pytest.mark.parametrize("c", [10.0, 1000.0])
def test_gamma_draw_matches_scipy_gamma(orc, c):
    from scipy import stats
    g = np.array([orc.gamma_draw(77, 5, i, 0x100, c) for i in range(20000)])
    p = stats.kstest(g, stats.gamma(c).cdf).pvalue
    assert p > 1e-3, p
    assert abs(g.mean() / c - 1.0) < 4.0 / math.sqrt(c * 20000)


def _base(orc, J=2, K=2, nf=8, index=5):
    cfg = small_cfg(J=J, K=K, ny=4, nv=4, nf=nf, P=64, index=index)
    sc = scenes.make_scene(cfg)
    return cfg, sc, orc.Oracle.from_scene(sc)


def test_predict_transitions(orc, OS):
    P, J = 4000, 2
    prm = OS.Params()
    x = np.zeros((P, 6))
    eta = np.full((J, P), 2.0e-3)
    s0 = OS.init_los(P, J, prm)
    s0.zeta = np.array([1.0, 0.0])
    s1 = OS.Slot(np.tile([-9.0, 0.0, 0.0], (P, 1)), np.full(P, 0.5 + 0.1j), np.full(P, 0.2), np.full(P, 0.6 / P),
                 np.array([0.3, 0.7]), 1)
    st = OS.State(x, eta, [s0, s1], n=3)
    xp, ep, sl = OS.predict(st, prm)
    r = ep / 2.0e-3
    assert abs(r.mean() - 1.0) < 4.0 * math.sqrt(0.1 / r.size)                 # E eta_n = eta_{n-1}
    assert abs(r.var() - 1.0 / prm.c_eta) < 0.1 / prm.c_eta                    # Var = eta^2 / c_eta
    assert np.allclose(sl[0].zeta, [prm.p_s_pr, prm.p_rev_pr], rtol=0, atol=1e-15)
    assert np.allclose(sl[1].zeta, prm.p_s_pr * s1.zeta + prm.p_rev_pr * (1 - s1.zeta), rtol=1e-15)
    assert np.allclose(sl[1].w, prm.p_s * s1.w, rtol=1e-15)
    d = sl[1].phi - s1.phi
    assert abs(d.std() / prm.sigma_sfv - 1.0) < 0.05                          # 4 mm SFV jitter
    dm = sl[1].mu - s1.mu
    assert abs(np.mean(np.abs(dm) ** 2) / prm.sigma_mu ** 2 - 1.0) < 0.06       # CN(0, sigma_mu^2)
    assert abs(np.mean(sl[1].gamma / s1.gamma) - 1.0) < 4.0 / math.sqrt(prm.c_gamma * P)
    assert sl[0].phi is None


def test_belief_vectors_closed_form(orc, OS):
    cfg, sc, o = _base(orc, J=2, K=1)
    P = 50
    x = np.tile(np.concatenate([scenes.P_TRUE, [0, 0, 0]]), (P, 1))
    rng = np.random.default_rng(2)
    w = rng.uniform(0.1, 1.0, P)
    w *= 0.7 / w.sum()
    mu, gam = 0.4 - 0.2j, 0.15
    los = OS.Slot(None, np.full(P, mu), np.full(P, gam), w, np.array([0.8, 0.6]), 0)
    wall = OS.Slot(np.tile(sc.sfv[0], (P, 1)), np.full(P, mu), np.full(P, gam), w, np.array([0.9, 0.5]), 1)
    for P_m in (P, 7):
        u, m, mw = OS.belief_vectors(o, x, [los, wall], P_m)
        for s, sl in enumerate([los, wall]):
            for j in range(cfg.J):
                st, psi = o.response(scenes.P_TRUE, j, s, sc.sfv)
                z, eps = sl.zeta[j], 0.7
                assert np.allclose(u[j, s], eps * mu * psi, rtol=1e-12, atol=1e-14)
                assert np.allclose(m[j, s], eps * z * math.sqrt(gam + abs(mu) ** 2 * (1 - z * eps)) * psi,
                                   rtol=1e-12, atol=1e-14)
                assert np.allclose(mw[j, s], eps * math.sqrt(gam + abs(mu) ** 2 * (1 - z)) * psi, rtol=1e-12,
                                   atol=1e-14)


def test_birth_weights_and_importance_ratios(orc, OS):
    from scipy import stats
    cfg, sc, o = _base(orc, J=2, K=2)
    y, eta = orc.measurement(o, sc, scenes.P_TRUE)
    P = 300
    prm = OS.Params(N_g=512, box=(-12.0, -5.0, -4.0, 14.0, 12.0, 4.0))
    st = OS.State(np.zeros((P, 6)), np.full((cfg.J, P), eta), [], n=2)
    b = OS.birth(o, st, prm, scenes.P_TRUE, y, np.zeros((0, 3)), 7)
    assert b is not None and b.ident == 7
    assert abs(b.w.sum() - prm.mu_b / (1 + prm.mu_b)) < 1e-14
    rc, _, _, mu_q, C, _ = o.birth_proposal(scenes.P_TRUE, np.zeros((0, 3)), y, prm.box, prm.N_g, prm.key, 2)
    Cj = C + 1e-12 * np.trace(C) * np.eye(3)
    lo, hi = np.array(prm.box[:3]), np.array(prm.box[3:])
    inside = np.all((b.phi >= lo) & (b.phi <= hi), axis=1)
    assert np.all(b.w[~inside] == 0.0)
    dens = stats.multivariate_normal(mu_q, Cj).pdf(b.phi[inside])
    r = b.w[inside] * dens                                                     # w ∝ 1 / f^p  =>  w f^p constant
    assert np.allclose(r, r[0], rtol=1e-8)
    assert np.all(np.abs(b.mu) <= prm.mu_max) and np.all((b.gamma >= 0) & (b.gamma <= prm.gamma_max))
    assert np.allclose(b.zeta, prm.p_b_pr)


def test_one_step_invariants_and_pruning(orc, OS):
    """A scene whose LOS and walls are known (PFs at the true SFVs and amplitudes, MT particles within 1 mm of the
    truth): the true PFs stay (existence > T_dec), a PF at a wrong SFV with a small prior existence is pruned."""
    cfg, sc, o = _base(orc, J=2, K=2)
    y, eta = orc.measurement(o, sc, scenes.P_TRUE)
    P = 64
    prm = OS.Params(P_m=64, N_g=512)
    rng = np.random.default_rng(0)
    x = np.zeros((P, 6))
    x[:, :3] = scenes.P_TRUE + 0.001 * rng.standard_normal((P, 3))
    full = lambda v: np.full(P, v)  # noqa: E731
    slots = [OS.Slot(None, full(sc.rho[0]), full(1e-3), full(1.0 / P), np.full(cfg.J, 0.9), 0)]
    for k in range(cfg.K):
        slots.append(OS.Slot(np.tile(sc.sfv[k], (P, 1)), full(sc.rho[k + 1]), full(1e-3), full(1.0 / P),
                             np.full(cfg.J, 0.9), k + 1))
    slots.append(OS.Slot(np.tile([30.0, 30.0, 0.0], (P, 1)), full(1e-4 + 0j), full(1e-4), full(0.02 / P),
                         np.full(cfg.J, 0.5), 3))
    phi_hat = {k + 1: sc.sfv[k] for k in range(cfg.K)}
    phi_hat[3] = np.array([30.0, 30.0, 0.0])
    st = OS.State(x, np.full((cfg.J, P), eta), slots, n=1, next_id=4, phi_hat=phi_hat)
    new, rep = OS.step(o, st, y, prm)
    assert rep["n_slots"] == 5                                                 # LOS, 2 walls, the weak PF, a birth
    for f, (logr, logM, ex) in zip(rep["features"], rep["pf"]):
        assert 0.0 <= f["exist"] <= 1.0 + 1e-12 and abs(f["exist"] - ex) < 1e-12
        assert np.all((f["zeta"] >= 0.0) & (f["zeta"] <= 1.0))
    ids = [s.ident for s in new.slots]
    assert ids[:3] == [0, 1, 2]                                                # the LOS and the true walls stay
    assert all(f["exist"] > prm.T_dec for f in rep["features"][:3])
    assert rep["features"][3]["exist"] < prm.T_pru and 3 not in ids            # pruned
    for s in new.slots:
        assert abs(s.w.sum() - next(f["exist"] for f in rep["features"] if f["ident"] == s.ident)) < 1e-12
    assert new.x.shape == (P, 6) and new.n == 2
    assert np.allclose(rep["w_eta"].sum(axis=1), 1.0, rtol=1e-12)
