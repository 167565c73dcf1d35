"""Pins of the oracle's F3 birth proposal: the residual projector, the coherent Bartlett spectrum
and the mode / moment matching, against numpy's pseudo-inverse, projector algebra, the Cauchy-Schwarz bound and
its equality case, coherent doubling over identical PAs, and zero mass."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2604_19723_b200 import scenes
from tests.helpers import tiny_scene

ORC_OK, ORC_EZEROMASS = 0, 3


def _setup(J=1, K=3, ny=4, nv=4, nf=16, wavefront="spherical", L=2):
    sc, cfg = tiny_scene(J=J, K=K, ny=ny, nv=nv, nf=nf)
    o = orc.Oracle.from_scene(sc, wavefront=wavefront)
    y, _ = orc.measurement(o, sc, scenes.P_TRUE, wavefront=wavefront)
    x_hat = scenes.P_TRUE + np.array([0.01, -0.02, 0.005])
    return sc, cfg, o, y.reshape(J, -1), x_hat, sc.sfv[:L]


def _psi_cols(o, x_hat, j, sfv_legacy):
    """Psi_j = [psi(x_hat, LOS) psi(x_hat, sfv_1) ...] from per-component responses (N_z x (L+1))."""
    cols = [o.response(x_hat, j, 0, sfv_legacy)[1]]
    for l in range(len(sfv_legacy)):
        st, p = o.response(x_hat, j, l + 1, sfv_legacy)
        assert st == 0
        cols.append(p)
    return np.stack(cols, axis=1)


@pytest.mark.parametrize("wavefront", ["spherical", "planar_wb", "planar_nb"])
def test_residual_matches_pinv(wavefront):
    sc, cfg, o, y, x_hat, sl = _setup(J=2, wavefront=wavefront)
    st, zr = o.birth_residual(x_hat, sl, y)
    assert st == ORC_OK
    for j in range(cfg.J):
        Psi = _psi_cols(o, x_hat, j, sl)
        ref = y[j] - Psi @ (np.linalg.pinv(Psi) @ y[j])
        assert np.max(np.abs(zr[j] - ref)) <= 1e-10 * np.linalg.norm(y[j])


def test_residual_projector_algebra():
    sc, cfg, o, y, x_hat, sl = _setup(J=1, L=3)
    st, zr = o.birth_residual(x_hat, sl, y)
    Psi = _psi_cols(o, x_hat, 0, sl)
    # orthogonal to the signal subspace, idempotent, and annihilates the subspace itself
    assert np.max(np.abs(Psi.conj().T @ zr[0])) <= 1e-10 * np.linalg.norm(Psi) * np.linalg.norm(y)
    st2, zr2 = o.birth_residual(x_hat, sl, zr)
    assert np.max(np.abs(zr2 - zr)) <= 1e-10 * np.linalg.norm(zr)
    a = np.array([1.0 + 0.5j, -0.3j, 0.2, 0.7 - 0.1j])
    st3, zr3 = o.birth_residual(x_hat, sl, (Psi @ a)[None])
    assert np.max(np.abs(zr3)) <= 1e-10 * np.linalg.norm(Psi @ a)


def test_bartlett_equality_case_closed_form():
    """LOS only (L = 0), z = psi(x_hat, p*), every candidate = p* (degenerate box): z~ = Pi_perp psi*, so
    P_B = |psi*^H Pi_perp psi*|^2 / Nz^2 = ||Pi_perp psi*||^4 / Nz^2 (Cauchy-Schwarz with equality)."""
    sc, cfg, o, y, x_hat, _ = _setup(J=1, L=0)
    p_star = sc.sfv[1]
    st, psi_star = o.response(x_hat, 0, 1, p_star[None])
    Psi = _psi_cols(o, x_hat, 0, np.zeros((0, 3)))
    r = psi_star - Psi @ (np.linalg.pinv(Psi) @ psi_star)
    box = np.concatenate([p_star, p_star])
    st, pb, cand, mu, C, ist = o.birth_proposal(x_hat, np.zeros((0, 3)), psi_star[None], box, 5, 3, 4)
    assert st == ORC_OK
    expect = np.linalg.norm(r) ** 4 / cfg.Nz ** 2
    assert np.allclose(pb, expect, rtol=1e-10)
    assert np.allclose(mu, p_star) and np.allclose(C, 0.0)


def test_bartlett_cauchy_schwarz_bound():
    sc, cfg, o, y, x_hat, sl = _setup(J=2)
    box = np.concatenate([sc.sfv[2] - 0.5, sc.sfv[2] + 0.5])
    st, pb, cand, mu, C, ist = o.birth_proposal(x_hat, sl, y, box, 64, 11, 0)
    assert st == ORC_OK
    st, zr = o.birth_residual(x_hat, sl, y)
    bound = (np.sum(np.linalg.norm(zr, axis=1)) / np.sqrt(cfg.Nz)) ** 2  # |sum_j <z~_j, psi>| <= sum_j ||z~_j|| ||psi||
    assert np.all(pb <= bound * (1 + 1e-12))


def test_bartlett_coherent_over_pas():
    """Two PAs with the same pose and the same snapshot: the coherent sum doubles the amplitude -> 4x power."""
    sc, cfg = tiny_scene(J=2, K=3)
    sc.pa_pos[1] = sc.pa_pos[0]
    sc.pa_rot[1] = sc.pa_rot[0]
    o2 = orc.Oracle.from_scene(sc)
    y2, _ = orc.measurement(o2, sc, scenes.P_TRUE)
    y2 = y2.reshape(2, -1)
    y2[1] = y2[0]
    o1 = orc.Oracle(sc.pa_pos[:1], sc.pa_rot[:1], cfg.ny, cfg.nv, sc.dy, sc.dv, cfg.f_pb(), cfg.fc, cfg.K)
    x_hat = scenes.P_TRUE + 0.01
    box = np.concatenate([sc.sfv[2] - 0.3, sc.sfv[2] + 0.3])
    st2, pb2, *_ = o2.birth_proposal(x_hat, sc.sfv[:1], y2, box, 32, 5, 1)
    st1, pb1, *_ = o1.birth_proposal(x_hat, sc.sfv[:1], y2[:1], box, 32, 5, 1)
    assert st1 == st2 == ORC_OK
    assert np.allclose(pb2, 4.0 * pb1, rtol=1e-10)


def test_birth_moments_and_candidates():
    sc, cfg, o, y, x_hat, sl = _setup(J=2, L=2)
    box = np.concatenate([sc.sfv[2] - 0.4, sc.sfv[2] + 0.4])
    st, pb, cand, mu, C, ist = o.birth_proposal(x_hat, sl, y, box, 200, 21, 9)
    assert st == ORC_OK
    assert ist == int(np.argmax(pb)) and np.array_equal(mu, cand[ist])
    assert np.all(cand >= box[:3]) and np.all(cand <= box[3:])
    for i in (0, 57, 199):
        assert np.array_equal(cand[i], orc.birth_candidate(21, 9, i, box))
    assert np.allclose(C, C.T) and np.min(np.linalg.eigvalsh(C)) >= -1e-15
    # the planted wall (in the residual: not a legacy component) dominates the spectrum near its position
    assert np.linalg.norm(mu - sc.sfv[2]) < 0.4


def test_birth_zero_mass():
    sc, cfg, o, y, x_hat, sl = _setup(J=1)
    box = np.concatenate([sc.sfv[2] - 0.4, sc.sfv[2] + 0.4])
    st, *_ = o.birth_proposal(x_hat, sl, np.zeros_like(y), box, 16, 1, 0)
    assert st == ORC_EZEROMASS
