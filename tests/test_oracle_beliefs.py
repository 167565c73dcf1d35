"""Oracle pins for rows A6-A9: normalization, moments, systematic resampling, RNG, prediction,
regularization, moment matching."""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy.special import logsumexp

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- A6 normalize
def test_normalize_sum_shift_uniform(orc):
    rng = np.random.default_rng(0)
    l = rng.normal(0, 50, 1000) - 1e5
    st, w, lse = orc.normalize(l)
    assert st == 0
    assert abs(w.sum() - 1.0) < 1e-12                              # weights sum to 1
    assert abs(lse - logsumexp(l)) < 1e-9 * abs(lse)              # library logsumexp
    st, w2, lse2 = orc.normalize(l + 1234.5)
    assert np.allclose(w, w2, rtol=1e-9, atol=1e-300)             # invariant to l + const
    st, w3, _ = orc.normalize(np.full(64, -7.0))
    assert np.allclose(w3, 1 / 64, rtol=1e-15)                    # uniform -> 1/P


def test_normalize_zero_mass_and_nan(orc):
    st, w, lse = orc.normalize(np.full(5, -np.inf))
    assert st == orc.EZEROMASS and lse == -np.inf
    st, w, lse = orc.normalize(np.array([0.0, np.nan]))
    assert st == orc.EINVAL


# ---------------------------------------------------------------- A7 moments
def test_moments_special_cases_and_numpy(orc):
    x = np.array([[1.0, 2, 3, 4, 5, 6]])
    st, est = orc.moments(x, np.ones(1))
    assert np.allclose(est[1:7], x[0]) and np.allclose(est[7:], 0.0)   # single particle -> itself
    x = np.array([[0.0, 0, 0, 1, 1, 1], [2.0, 4, -2, 3, 1, -1]])
    st, est = orc.moments(x, np.array([0.5, 0.5]))
    assert np.allclose(est[1:7], x.mean(0))                              # symmetric pair -> midpoint
    rng = np.random.default_rng(1)
    x = rng.normal(size=(500, 6))
    w = rng.uniform(size=500)
    w /= w.sum()
    st, est = orc.moments(x, w)
    mean = np.average(x, axis=0, weights=w)
    cov = np.cov(x.T, aweights=w, bias=True)
    iu = np.triu_indices(6)
    assert np.allclose(est[1:7], mean, atol=1e-14)
    assert np.allclose(est[7:], cov[iu], atol=1e-14)


# ---------------------------------------------------------------- A8 resampling
def counts(anc, n):
    return np.bincount(anc, minlength=n)


def test_resampling_hand_trace(orc):
    g = json.load(open(os.path.join(GOLDEN, "resampling_hand_trace.json")))
    for case in g["cases"]:
        w = np.zeros(case["P_out"])
        w[:3] = case["w"]
        st, anc = orc.resample(w, case["u_bits"])
        assert st == 0
        assert list(counts(anc, 10)[:3]) == case["counts"]


def test_resampling_uniform_onehot_bounds(orc):
    P = 257
    st, anc = orc.resample(np.full(P, 1.0 / P), 2**31)
    assert np.array_equal(anc, np.arange(P))                          # uniform -> each once
    w = np.zeros(P)
    w[100] = 1.0
    st, anc = orc.resample(w, 99)
    assert np.all(anc == 100)                                          # one-hot -> all copies
    rng = np.random.default_rng(2)
    for _ in range(50):
        w = rng.exponential(size=P) * (rng.uniform(size=P) < 0.7)
        st, anc = orc.resample(w, int(rng.integers(0, 2**32)))
        c = counts(anc, P)
        q = w / w.sum()
        assert np.all(c >= np.floor(P * q) - 1e-9) and np.all(c <= np.ceil(P * q) + 1e-9)
        assert np.all(c[w == 0] == 0)                                  # q = 0 never drawn
        assert np.all(np.diff(anc) >= 0)                               # ancestors sorted


def alg2_float(w, u):
    """Arulampalam et al. Alg. 2 in floating point: u_1 = u/P, u_i = u_1 + (i-1)/P, i++ while
    u_i > c_i (cumulative normalized weights)."""
    P = len(w)
    c = np.cumsum(w / w.sum())
    out = np.empty(P, dtype=np.int64)
    i = 0
    for jj in range(P):
        uj = (u + jj) / P
        while uj > c[i] and i < P - 1:
            i += 1
        out[jj] = i
    return out


def test_resampling_equals_float_alg2(orc):
    rng = np.random.default_rng(3)
    for trial in range(20):
        P = int(rng.integers(5, 400))
        w = rng.exponential(size=P)
        u_bits = int(rng.integers(1, 2**32))
        st, anc = orc.resample(w, u_bits)
        ref = alg2_float(w, u_bits / 2**32)
        assert np.array_equal(anc, ref)


# ---------------------------------------------------------------- RNG
def test_philox_kat(orc):
    g = json.load(open(os.path.join(GOLDEN, "philox4x32_10_kat.json")))
    for v in g["vectors"]:
        out = orc.philox([int(x, 16) for x in v["ctr"]], [int(x, 16) for x in v["key"]])
        assert out == [int(x, 16) for x in v["out"]]


def test_box_muller_from_philox(orc):
    key, step, idx, stream = 0x1234_5678_9ABC_DEF0, 7, 123456789, 2
    x = orc.philox([idx & 0xFFFFFFFF, idx >> 32, step, stream], [key & 0xFFFFFFFF, key >> 32])
    u = [(xi + 0.5) / 2**32 for xi in x]
    r0, r1 = math.sqrt(-2 * math.log(u[0])), math.sqrt(-2 * math.log(u[2]))
    ref = [r0 * math.cos(2 * math.pi * u[1]), r0 * math.sin(2 * math.pi * u[1]),
           r1 * math.cos(2 * math.pi * u[3]), r1 * math.sin(2 * math.pi * u[3])]
    assert np.allclose(orc.normals4(key, step, idx, stream), ref, rtol=1e-14)


# ---------------------------------------------------------------- A9 predict / regularize
def test_predict_ncv(orc):
    rng = np.random.default_rng(4)
    x = rng.normal(size=(100, 6))
    T = 0.1
    F = np.eye(6)
    F[0, 3] = F[1, 4] = F[2, 5] = T                                    # NCV F
    out = orc.predict(x, 0, T, 0.0, 5, 1)
    assert np.allclose(out, x @ F.T, atol=1e-15)                       # sigma_v = 0 -> F x
    n = 40000
    out = orc.predict(np.zeros((n, 6)), 0, T, 0.5, 5, 1)
    G = np.vstack([T * T / 2 * np.eye(3), T * np.eye(3)])
    Q = 0.25 * G @ G.T                                                 # sigma_v^2 Gamma Gamma^T
    emp = out.T @ out / n
    assert np.allclose(emp, Q, atol=0.05 * Q.max())


def test_regularize(orc):
    hval = (4 / (8 * 1000)) ** 0.1
    assert abs(hval - 0.46763) < 1e-4                                  # h_opt for d=6, P=1000
    x = np.random.default_rng(5).normal(size=(10, 6))
    out = orc.regularize(x, 0, 1000, np.zeros(21), 1, 2)
    assert np.allclose(out, x)                                         # zero covariance -> identity
    A = np.random.default_rng(6).normal(size=(6, 6))
    Sig = A @ A.T / 6
    iu = np.triu_indices(6)
    n = 40000
    out = orc.regularize(np.zeros((n, 6)), 0, n, Sig[iu], 3, 4)
    h = (4 / (8 * n)) ** 0.1
    emp = out.T @ out / n
    assert np.allclose(emp, h * h * Sig, atol=0.05 * h * h * np.abs(Sig).max())


# ---------------------------------------------------------------- moment matching
def test_moment_match_enumeration(orc):
    # Bernoulli(eps) x Bernoulli(zeta) x CN(mu, gamma): enumerate the 2^2 existence
    # configurations (Prop. 1 setting); compare exact mean / variance (C-amb-7)
    for eps, zeta, gamma, mu in [(0.7, 0.9, 0.2, 0.8 * np.exp(0.3j)), (1.0, 1.0, 0.5, 1 + 1j),
                                 (0.3, 0.5, 0.0, -0.2j), (0.0, 0.5, 1.0, 1.0)]:
        mean, second = 0.0, 0.0
        for r, rp in itertools.product([0, 1], [0, 1]):
            pr = (eps if r else 1 - eps) * (zeta if rp else 1 - zeta)
            on = r * rp
            mean += pr * on * mu
            second += pr * on * (gamma + abs(mu) ** 2)
        var = second - abs(mean) ** 2
        m, v = orc.moment_match(mu, gamma, eps * zeta)
        assert abs(m - mean) < 1e-15 and abs(v - var) < 1e-14


# ---------------------------------------------------------------- A8 in the BP step: masses e^{l - M} (C-amb-23)
def test_resample_loglik_hand_trace(orc):
    """S:L414's trace with the weights given as log-weights: l = ln w (+ an offset that makes M != 0)."""
    g = json.load(open(os.path.join(GOLDEN, "resampling_hand_trace.json")))
    for case in g["cases"]:
        l = np.full(case["P_out"], -np.inf)
        l[:3] = np.log(case["w"]) - 4321.0
        st, anc = orc.resample_loglik(l, case["u_bits"])
        assert st == 0
        assert list(counts(anc, 10)[:3]) == case["counts"]


def test_resample_loglik_equals_resample_of_exp(orc):
    """r_p = e^{l_p - M} has max exactly e^0 = 1, so orc_resample (w / w_max, pinned above) applied to the vector r
    (formed here with the C library's exp through math.exp) must give the same ancestors bit for bit."""
    rng = np.random.default_rng(9)
    for trial in range(30):
        P = int(rng.integers(1, 3000))
        l = rng.normal(-2e4, 40.0, P)
        l[rng.uniform(size=P) < 0.1] = -np.inf
        if not np.isfinite(l).any():
            l[0] = 0.0
        M = np.max(l)
        r = np.array([math.exp(v - M) if np.isfinite(v) else 0.0 for v in l])
        u = int(rng.integers(0, 2**32))
        st1, a1 = orc.resample_loglik(l, u)
        st2, a2 = orc.resample(r, u)
        assert st1 == 0 and st2 == 0
        assert np.array_equal(a1, a2)


def test_resample_loglik_bounds_and_errors(orc):
    rng = np.random.default_rng(10)
    P = 511
    for _ in range(20):
        l = rng.normal(0, 3, P)
        st, anc = orc.resample_loglik(l, int(rng.integers(0, 2**32)))
        q = np.exp(l - l.max())
        q /= q.sum()
        c = counts(anc, P)
        assert np.all(c >= np.floor(P * q) - 1) and np.all(c <= np.ceil(P * q) + 1)   # quantization: +-1 slack
        assert np.all(np.diff(anc) >= 0)
    assert orc.resample_loglik(np.full(4, -np.inf), 1)[0] == orc.EZEROMASS
    assert orc.resample_loglik(np.array([0.0, np.nan]), 1)[0] == orc.EINVAL


def test_step_update_composition(orc):
    """orc_step_update follows the paper's order: normalize -> MMSE moments of the weighted set
     -> systematic resampling with u of the step -> gather -> regularization with the
    pre-resampling covariance.  Composed here from the separately pinned oracle pieces."""
    rng = np.random.default_rng(12)
    P = 777
    x = rng.normal(size=(P, 6))
    l = rng.normal(-5e3, 2.0, P)
    key, step = 0xABCDEF12345, 4
    st, xo, est, lse, anc = orc.step_update(l, x, key, step)
    assert st == 0
    st, w, lse_ref = orc.normalize(l)
    st, est_ref = orc.moments(x, w)
    st, a_ref = orc.resample_loglik(l, orc.step_u_bits(key, step))
    xr = orc.regularize(x[a_ref], 0, P, est_ref[7:], key, step)
    assert lse == lse_ref and np.array_equal(est, est_ref) and np.array_equal(anc, a_ref)
    assert np.array_equal(xo, xr)
    st, xo2, _, _, _ = orc.step_update(l, x, key, step, regularize=False)
    assert np.array_equal(xo2, x[a_ref])


def test_bp_step_is_predict_loglik_update(orc):
    """orc_bp_step = predict -> l -> orc_step_update."""
    from paper_2604_19723_b200 import scenes
    from tests.helpers import small_cfg
    cfg = small_cfg(J=1, K=1, ny=2, nv=2, nf=8, P=200)
    sc = scenes.make_scene(cfg)
    o = orc.Oracle.from_scene(sc)
    y, eta = orc.measurement(o, sc, scenes.P_TRUE)
    m, v = scenes.priors(sc, "nzm")
    eta = np.full(cfg.J, eta)
    x = scenes.make_particles(cfg)
    st, xb, estb, lseb, ancb = o.bp_step(x, sc.sfv, y, m, v, eta, 0.1, 0.5, 77, 3)
    assert st == 0
    xp = orc.predict(x, 0, 0.1, 0.5, 77, 3)
    st, l = o.loglik(xp, sc.sfv, y, m, v, eta)
    st, xu, estu, lseu, ancu = orc.step_update(l, xp, 77, 3)
    assert np.array_equal(xb, xu) and np.array_equal(estb, estu) and lseb == lseu and np.array_equal(ancb, ancu)
