"""Oracle pins for the coherent likelihood rows A3-A5."""
import math

import numpy as np
import pytest

from paper_2604_19723_b200 import scenes
from tests.helpers import tiny_scene


def dense_logcn(z, mu, Cm):
    """Plain definition log CN(z; mu, C) = -N ln pi - ln det C - (z-mu)^H C^-1 (z-mu) (numpy)."""
    e = z - mu
    sign, logdet = np.linalg.slogdet(Cm)
    quad = np.real(np.conj(e) @ np.linalg.solve(Cm, e))
    return -len(z) * math.log(math.pi) - logdet - quad


def dense_particle(o, p, sfv, y, m, v, eta):
    tot = 0.0
    for j in range(o.J):
        Psi = o.responses(p, j, sfv)
        z = y[j].reshape(-1)
        Cm = eta[j] * np.eye(o.Nz) + (Psi * v[j][None, :]) @ np.conj(Psi.T)
        tot += dense_logcn(z, Psi @ m[j], Cm)
    return tot


def setup(orc, J=1, K=2, ny=4, nv=4, nf=16, wavefront="spherical", pathloss=False, mode="nzm",
          n=8, index=91):
    sc, cfg = tiny_scene(J=J, K=K, ny=ny, nv=nv, nf=nf, index=index)
    o = orc.Oracle.from_scene(sc, wavefront=wavefront, pathloss=pathloss)
    y, eta = orc.measurement(o, sc, scenes.P_TRUE)
    m, v = scenes.priors(sc, mode)
    eta_j = np.full(J, eta)
    x = scenes.make_particles(scenes.custom_config("t", J=J, K=K, ny=ny, nv=nv, nf=nf, P=n, index=index))
    x[0, :3] = scenes.P_TRUE
    return o, sc, y, m, v, eta_j, x


@pytest.mark.parametrize("wf,pl,J,K,mode", [
    ("spherical", False, 1, 2, "nzm"),
    ("spherical", False, 2, 3, "zm"),
    ("planar_wb", False, 1, 2, "nzm"),
    ("planar_nb", True, 2, 1, "nzm"),
    ("spherical", True, 1, 0, "nzm"),
])
def test_woodbury_equals_dense_definition(orc, wf, pl, J, K, mode):
    # S-V-C fast form == dense N_z x N_z log-density
    o, sc, y, m, v, eta, x = setup(orc, J=J, K=K, wavefront=wf, pathloss=pl, mode=mode)
    if pl:
        v = v * 1e4  # path-loss-compensated responses are ~1e-3: rescale the prior variance
        m = m * 100
    st, l = o.loglik(x, sc.sfv, y, m, v, eta)
    assert st == 0
    # with path loss, cond(C) ~ v Nz / eta ~ 1e7: the dense numpy side loses ~7 digits
    tol = 1e-8 if pl else 1e-10
    for i in range(x.shape[0]):
        d = dense_particle(o, x[i, :3], sc.sfv, y, m, v, eta)
        assert abs(l[i] - d) <= tol * abs(d), (i, l[i], d)


def test_zero_prior_variance_entry(orc):
    o, sc, y, m, v, eta, x = setup(orc, K=3)
    v = v.copy()
    v[0, 2] = 0.0
    st, l = o.loglik(x, sc.sfv, y, m, v, eta)
    for i in range(3):
        d = dense_particle(o, x[i, :3], sc.sfv, y, m, v, eta)
        assert abs(l[i] - d) <= 1e-10 * abs(d)


def test_sherman_morrison_single_component(orc):
    # S = 1: l = -Nz ln(pi eta) - ln(1 + v Nz/eta) - [||e||^2 - v |psi^H e|^2/(eta + v Nz)]/eta
    # (matrix inversion lemma)
    o, sc, y, m, v, eta, x = setup(orc, K=0)
    st, l = o.loglik(x, sc.sfv, y, m, v, eta)
    for i in range(x.shape[0]):
        psi = o.responses(x[i, :3], 0, sc.sfv)[:, 0]
        z = y[0].reshape(-1)
        e = z - m[0, 0] * psi
        vv, et, N = v[0, 0], eta[0], o.Nz
        ref = (-N * math.log(math.pi * et) - math.log(1 + vv * N / et)
               - (np.vdot(e, e).real - vv * abs(np.vdot(psi, e)) ** 2 / (et + vv * N)) / et)
        assert abs(l[i] - ref) <= 1e-11 * abs(ref)


def test_v_zero_limit(orc):
    # v -> 0: l -> -Nz ln(pi eta) - ||z - Psi m||^2/eta
    o, sc, y, m, v, eta, x = setup(orc, K=2, J=2)
    v0 = np.zeros_like(v)
    st, l = o.loglik(x, sc.sfv, y, m, v0, eta)
    for i in range(x.shape[0]):
        ref = 0.0
        for j in range(2):
            Psi = o.responses(x[i, :3], j, sc.sfv)
            e = y[j].reshape(-1) - Psi @ m[j]
            ref += -o.Nz * math.log(math.pi * eta[j]) - np.vdot(e, e).real / eta[j]
        assert abs(l[i] - ref) <= 1e-12 * abs(ref)


def test_amplitude_lmmse_and_least_squares_limit(orc):
    # a = m + V Psi^H C^-1 (z - Psi m) (LMMSE); v -> inf: a -> G^-1 c (Type-I fit)
    o, sc, y, m, v, eta, x = setup(orc, K=2)
    st, l, amp = o.loglik(x[:3], sc.sfv, y, m, v, eta, want_amp=True)
    for i in range(3):
        Psi = o.responses(x[i, :3], 0, sc.sfv)
        z = y[0].reshape(-1)
        Cm = eta[0] * np.eye(o.Nz) + (Psi * v[0][None, :]) @ np.conj(Psi.T)
        ref = m[0] + v[0] * (np.conj(Psi.T) @ np.linalg.solve(Cm, z - Psi @ m[0]))
        assert np.allclose(amp[i, 0], ref, rtol=1e-9, atol=1e-12)
    vbig = np.full_like(v, 1e10)
    st, l, amp = o.loglik(x[:3], sc.sfv, y, m, vbig, eta, want_amp=True)
    for i in range(3):
        Psi = o.responses(x[i, :3], 0, sc.sfv)
        z = y[0].reshape(-1)
        ls = np.linalg.solve(np.conj(Psi.T) @ Psi, np.conj(Psi.T) @ z)
        assert np.allclose(amp[i, 0], ls, rtol=1e-5, atol=1e-7)


def test_coherence_and_permutation_invariance(orc):
    # (z, m) -> (e^{j theta} z, e^{j theta} m) leaves l unchanged (coherent premise);
    # permuting the components leaves l unchanged
    o, sc, y, m, v, eta, x = setup(orc, K=3, J=2)
    st, l = o.loglik(x, sc.sfv, y, m, v, eta)
    rot = np.exp(1j * 0.73)
    st, l2 = o.loglik(x, sc.sfv, y * rot, m * rot, v, eta)
    assert np.allclose(l, l2, rtol=1e-12)
    perm = [0, 3, 1, 2]  # LOS stays first; walls permuted
    sfv_p = sc.sfv[[p - 1 for p in perm[1:]]]
    st, l3 = o.loglik(x, sfv_p, y, m[:, perm], v[:, perm], eta)
    assert np.allclose(l, l3, rtol=1e-12)


def test_matched_filter_peak(orc):
    # noise-free z = rho psi(p*), S = 1, m = 0 => l(p) <= l(p*) on any grid (Cauchy-Schwarz)
    sc, cfg = tiny_scene(K=0, index=93)
    o = orc.Oracle.from_scene(sc)
    pstar = scenes.P_TRUE
    z = 0.8 * np.exp(0.4j) * o.responses(pstar, 0, sc.sfv)[:, 0]
    y = z.reshape(1, o.nf, o.Na)
    g = np.stack(np.meshgrid(np.linspace(-0.2, 0.2, 7), np.linspace(-0.2, 0.2, 7), [0.0]), -1).reshape(-1, 3)
    x = pstar[None, :] + g
    st, l = o.loglik(np.vstack([pstar[None], x]), sc.sfv, y, np.zeros((1, 1)), np.ones((1, 1)), np.ones(1) * 0.01)
    assert np.all(l[1:] <= l[0] + 1e-9 * abs(l[0]))


def test_terms_gram_closed_form_and_invariants(orc):
    # G_ss = Nz, G Hermitian PSD; G_ab = sum_m e^{j 2 pi (d_a,m - d_b,m) fc/c} D_N((d_a,m - d_b,m) df/c)
    # on the symmetric uniform grid (geometric series; P:L769 fn), distances from the independent
    # reflection construction; c = Psi^H z
    from tests.helpers import reflect
    o, sc, y, m, v, eta, x = setup(orc, K=3, J=2, ny=3, nv=4, nf=24)
    st, c, G = o.terms(x[:4], sc.sfv, y)
    assert st == 0
    cfg_f = o.f_pb
    fc, df, N = sc.cfg.fc, cfg_f[1] - cfg_f[0], o.nf
    C = 299_792_458.0
    pt = o.template()
    for i in range(4):
        p = x[i, :3]
        for j in range(2):
            Gj = G[i, j]
            assert np.allclose(np.diag(Gj).real, o.Nz, rtol=1e-13)
            assert np.allclose(Gj, Gj.conj().T, atol=1e-9)
            assert np.linalg.eigvalsh(Gj).min() > -1e-8 * o.Nz
            cols0 = sc.pa_pos[j][:, None] + sc.pa_rot[j] @ pt
            d = []
            for s in range(o.S):
                cols = cols0 if s == 0 else np.stack([reflect(cols0[:, mm], sc.sfv[s - 1]) for mm in range(o.Na)], 1)
                d.append(np.linalg.norm(p[:, None] - cols, axis=0))
            for a in range(o.S):
                for b in range(o.S):
                    if a == b:
                        continue
                    dd = d[a] - d[b]
                    xx = dd * df / C
                    D = np.sin(np.pi * N * xx) / np.sin(np.pi * xx)
                    ref = np.sum(np.exp(2j * np.pi * dd * fc / C) * D)
                    assert abs(Gj[a, b] - ref) <= 1e-9 * o.Nz
            Psi = o.responses(p, j, sc.sfv)
            assert np.allclose(c[i, j], Psi.conj().T @ y[j].reshape(-1), rtol=1e-12, atol=1e-9)


def test_sfv_per_particle_matches_shared(orc):
    # paired SFVs (C-amb-8): [P][K][3] with identical rows == shared [K][3]
    o, sc, y, m, v, eta, x = setup(orc, K=2)
    st, l = o.loglik(x, sc.sfv, y, m, v, eta)
    pp = np.broadcast_to(sc.sfv[None], (x.shape[0], 2, 3)).copy()
    st, l2 = o.loglik(x, pp, y, m, v, eta, sfv_per_particle=True)
    assert np.array_equal(l, l2)


def test_logw_prior_and_degenerate(orc):
    o, sc, y, m, v, eta, x = setup(orc, K=1)
    lw = np.linspace(-3, 1, x.shape[0])
    st, l = o.loglik(x, sc.sfv, y, m, v, eta)
    st, l2 = o.loglik(x, sc.sfv, y, m, v, eta, logw_prior=lw)
    assert np.allclose(l2 - l, lw, atol=1e-9)
    x2 = x.copy()
    x2[1, :3] = sc.pa_pos[0]  # MT on the PA phase centre
    st, l3 = o.loglik(x2, sc.sfv, y, m, v, eta)
    assert st == orc.EDEGENERATE and l3[1] == -np.inf and np.isfinite(l3[0])
