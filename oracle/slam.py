"""F4 oracle: one time step of the synthetic direct-MP-SLAM BP method, written out in the paper's order.

TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline / reference legs).  Plain numpy
around the fp64 C oracle (oracle/cdms_oracle.c); no blocking, fusion or reordering beyond the paper's schedule.

Schedule: (i) prediction messages of every state from time n-1 -- MT (NCV), noise (Gamma), legacy PFs
(survival + Gaussian / Gamma transitions), PPRs (survival / revival) -- and the birth message of one new PF (Q = 1,
P:L3257-3346); (ii)-(iii) flooding: every update message from the same prediction messages -- iota~ (MT), nu~ (noise),
kappa~ (each PF), omega~ (each PPR); then beliefs, systematic resampling, regularization of
the MT belief and of the PFs' SFV particles, MMSE estimates, declaration and pruning.  The readings F4a-F4k of
DESIGN.md section 3 fix what the paper leaves open; each is cited where it is used.

Random numbers: counter-based Philox4x32-10 blocks (key; index, index >> 32, n, stream) -- the same counters as the
CUDA driver, which implements the same generator itself (no shared code):
  stream 0 MT prediction normals, 1-2 MT regularization, 3 MT resampling offset (rows A8, A9);
  0x100 + 16 j + a: noise Gamma draw of PA j, attempt a;     0x200 + 16 i: SFV jitter normals of slot i;
  0x201 + 16 i: amplitude-mean jitter normals of slot i;       0x300 + 16 i + a: amplitude-variance Gamma of slot i;
  0x400 + i: resampling offset of slot i's PF;                  0x500 + j: resampling offset of PA j's noise;
  0x600 / 0x601: birth SFV normals / birth amplitude uniforms; 0x700 + 16 i: SFV regularization normals of slot i;
  birth candidates: orc_birth_candidate, counter n.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

from oracle import oracle as O

S_MAX = 9          # LOS + 8 PFs: the likelihood's component limit
ST_NOISE, ST_SFV, ST_MU, ST_GAMMA, ST_PF_RES, ST_NOISE_RES, ST_BIRTH_N, ST_BIRTH_U, ST_PF_REG = (
    0x100, 0x200, 0x201, 0x300, 0x400, 0x500, 0x600, 0x601, 0x700)


@dataclasses.dataclass
class Params:
    """Transition, birth and threshold constants of Experiment 1."""
    T: float = 0.1                 # NCV time step (C-amb-17)
    sigma_v: float = 0.5           # NCV process noise (m/s^2)
    c_eta: float = 10.0            # noise variance Gamma constant
    c_gamma: float = 1000.0        # amplitude variance Gamma constant
    sigma_mu: float = 0.03         # amplitude mean CN std
    sigma_sfv: float = 0.004       # SFV jitter std, 4 mm
    p_s: float = 0.8               # PF survival
    p_s_pr: float = 0.9            # PPR survival
    p_rev_pr: float = 0.1          # PPR revival
    p_b_pr: float = 0.9            # PPR birth
    mu_b: float = 0.5              # Poisson birth mean, Q = 1
    gamma_max: float = 5.0         # birth hyperprior U(0, gamma_max)
    mu_max: float = 0.001          # birth hyperprior U(|mu| <= mu_max)
    T_dec: float = 0.5             # declaration threshold
    T_pru: float = 0.1             # pruning threshold
    box: tuple = (-7.0, -2.0, -2.0, 9.0, 9.0, 2.0)   # SFV birth box [2 p_min, 2 p_max]
    N_g: int = 4096                # birth-proposal candidates (F3)
    P_m: int = 256                 # belief-average sample size (reading F4c)
    key: int = 1234                # Philox key
    regularize: bool = True        # MT and PF-SFV regularization


@dataclasses.dataclass
class Slot:
    """One PF (slot 0 = the LOS s = 0, phi None): particles paired with the MT particles by index (C-amb-8)."""
    phi: Optional[np.ndarray]      # [P][3] SFV particles (None for the LOS)
    mu: np.ndarray                 # [P] complex amplitude means
    gamma: np.ndarray              # [P] amplitude variances
    w: np.ndarray                  # [P] PF weights, sum = existence probability (eq. existenceProb)
    zeta: np.ndarray               # [J] PPR existence probabilities
    ident: int = 0


@dataclasses.dataclass
class State:
    x: np.ndarray                  # [P][6] MT particles (equal weights after resampling)
    eta: np.ndarray                # [J][P] noise-variance particles (equal weights)
    slots: list                    # [Slot]
    n: int = 1                     # the time index of the NEXT step
    next_id: int = 1
    phi_hat: Optional[dict] = None  # ident -> previous MMSE SFV (birth proposal's legacy SFVs)


def philox_u32(key, index, step, stream):
    return O.philox([index & 0xFFFFFFFF, index >> 32, step, stream], [key & 0xFFFFFFFF, key >> 32])


def _oracle_for(base, K):
    return O.Oracle(base.pa_pos, base.pa_rot, base.ny, base.nv, base.sc.dy, base.sc.dv, base.f_pb, base.sc.fc, K,
                    wavefront=base.wavefront)


def _psi(orc, x, j, phi):
    """psi^(j)(x, phi): the LOS (phi None, component 0) or the wall of SFV phi (component 1)."""
    if phi is None:
        st, v = orc.response(x, j, 0, np.zeros((1, 3)))
    else:
        st, v = orc.response(x, j, 1, np.asarray(phi).reshape(1, 3))
    if st:
        raise ValueError(f"response status {st}")
    return v


def init_los(P, J, prm: Params):
    """The LOS PF at n = 0, introduced 'the same way as new PFs': amplitude hyperpriors, weights p_B / P,
    PPR probabilities p_B^PR (reading F4j)."""
    mu = np.zeros(P, dtype=complex)
    gam = np.zeros(P)
    for p in range(P):
        u = philox_u32(prm.key, p, 0, ST_BIRTH_U)
        u0, u1, u2 = [(u[i] + 0.5) * 2.0 ** -32 for i in range(3)]
        mu[p] = prm.mu_max * math.sqrt(u0) * complex(math.cos(2 * math.pi * u1), math.sin(2 * math.pi * u1))
        gam[p] = prm.gamma_max * u2
    pb = prm.mu_b / (1.0 + prm.mu_b)
    return Slot(None, mu, gam, np.full(P, pb / P), np.full(J, prm.p_b_pr), 0)


def predict(st: State, prm: Params):
    """Phase (i): prediction messages (transitions P:L3757-3815)."""
    n, key = st.n, prm.key
    P = st.x.shape[0]
    J = st.eta.shape[0]
    x = O.predict(st.x, 0, prm.T, prm.sigma_v, key, n)                     # beta: NCV draw, w_beta = 1/P
    eta = st.eta.copy()
    for j in range(J):                                                     # xi: Gamma(c_eta, eta / c_eta)
        for p in range(P):
            eta[j, p] *= O.gamma_draw(key, n, p, ST_NOISE + 16 * j, prm.c_eta) / prm.c_eta
    slots = []
    for i, s in enumerate(st.slots):                                       # alpha (legacy): p_s w, transitions
        phi = None if s.phi is None else s.phi.copy()
        mu, gam = s.mu.copy(), s.gamma.copy()
        for p in range(P):
            if phi is not None:
                nn = O.normals4(key, n, p, ST_SFV + 16 * i)
                phi[p] += prm.sigma_sfv * nn[:3]
            nm = O.normals4(key, n, p, ST_MU + 16 * i)
            mu[p] += prm.sigma_mu * complex(nm[0], nm[1]) / math.sqrt(2.0)   # CN(0, sigma_mu^2)
            gam[p] *= O.gamma_draw(key, n, p, ST_GAMMA + 16 * i, prm.c_gamma) / prm.c_gamma
        zeta = prm.p_s_pr * s.zeta + prm.p_rev_pr * (1.0 - s.zeta)         # zeta: survival / revival
        slots.append(Slot(phi, mu, gam, prm.p_s * s.w, zeta, s.ident))
    return x, eta, slots


def stats(slot: Slot):
    """(existence eps, mean mu, mean gamma, mean phi) of a PF particle representation (weights sum to eps)."""
    eps = float(np.sum(slot.w))
    if eps <= 0.0:
        return 0.0, 0j, 0.0, None
    mu = complex(np.sum(slot.w * slot.mu) / eps)
    gam = float(np.sum(slot.w * slot.gamma) / eps)
    phi = None if slot.phi is None else np.sum(slot.w[:, None] * slot.phi, axis=0) / eps
    return eps, mu, gam, phi


def birth(orc, st: State, prm: Params, x_pred_hat, y, legacy_phi, ident):
    """Birth message of the new PF (Q = 1): F3 proposal N(mu_q, C_q), particles phi_p ~ N(mu_q, C_q),
    amplitude hyperpriors, importance weights f_B / f_B^p normalized to p_B (reading F4h)."""
    P = st.x.shape[0]
    J = orc.J
    sl = np.asarray(legacy_phi).reshape(-1, 3)
    rc, _, _, mu_q, C, _ = orc.birth_proposal(x_pred_hat, sl, y, prm.box, prm.N_g, prm.key, st.n)
    if rc:
        return None
    Cj = C + 1e-12 * np.trace(C) * np.eye(3)
    try:
        L = np.linalg.cholesky(Cj)
    except np.linalg.LinAlgError:
        return None
    lo, hi = np.asarray(prm.box[:3]), np.asarray(prm.box[3:])
    phi = np.zeros((P, 3))
    mu = np.zeros(P, dtype=complex)
    gam = np.zeros(P)
    lw = np.full(P, -np.inf)
    for p in range(P):
        nn = O.normals4(prm.key, st.n, p, ST_BIRTH_N)
        phi[p] = mu_q + L @ nn[:3]
        u = philox_u32(prm.key, p, st.n, ST_BIRTH_U)
        u0, u1, u2 = [(u[i] + 0.5) * 2.0 ** -32 for i in range(3)]
        mu[p] = prm.mu_max * math.sqrt(u0) * complex(math.cos(2 * math.pi * u1), math.sin(2 * math.pi * u1))
        gam[p] = prm.gamma_max * u2
        if np.all(phi[p] >= lo) and np.all(phi[p] <= hi):                 # f_B = U(box): constant inside
            lw[p] = 0.5 * float(nn[0] ** 2 + nn[1] ** 2 + nn[2] ** 2)      # 1 / N(phi_p; mu_q, C) up to a constant
    if not np.isfinite(np.max(lw)):
        return None
    wt = np.exp(lw - np.max(lw))
    pb = prm.mu_b / (1.0 + prm.mu_b)
    return Slot(phi, mu, gam, pb * wt / np.sum(wt), np.full(J, prm.p_b_pr), ident)


def belief_vectors(orc, x, slots, P_m):
    """Per slot s and PA j the belief averages over paired particles (reading F4c; P:L686-698, P:L838-846,
    eq. musnj3/4): u = eps sum_k pi_k mu_k psi_k (mu~_4; mu~_3 = zeta u), m = eps zeta sum_k pi_k sqrt(gamma_k +
    |mu_k|^2 (1 - zeta eps)) psi_k, m_omega = eps sum_k pi_k sqrt(gamma_k + |mu_k|^2 (1 - zeta)) psi_k, on the
    sample p_k = floor((2k+1) P / (2K)), K = min(P, P_m), pi_k = w_{p_k} / sum_k w_{p_k}."""
    P = x.shape[0]
    J, Nz = orc.J, orc.Nz
    K = min(P, P_m)
    idx = [((2 * k + 1) * P) // (2 * K) for k in range(K)]
    S = len(slots)
    u = np.zeros((J, S, Nz), dtype=complex)
    m = np.zeros((J, S, Nz), dtype=complex)
    mw = np.zeros((J, S, Nz), dtype=complex)
    for s, sl in enumerate(slots):
        eps = float(np.sum(sl.w))
        ws = sl.w[idx]
        if eps <= 0.0 or np.sum(ws) <= 0.0:
            continue
        pi = ws / np.sum(ws)
        for j in range(J):
            z = sl.zeta[j]
            for k, p in enumerate(idx):
                psi = _psi(orc, x[p, :3], j, None if sl.phi is None else sl.phi[p])
                a2 = abs(sl.mu[p]) ** 2
                u[j, s] += eps * pi[k] * sl.mu[p] * psi
                m[j, s] += eps * z * pi[k] * math.sqrt(sl.gamma[p] + a2 * (1.0 - z * eps)) * psi
                mw[j, s] += eps * pi[k] * math.sqrt(sl.gamma[p] + a2 * (1.0 - z)) * psi
    return u, m, mw


def regularize_sfv(phi_res, phi, w, phi_hat, prm: Params, n, s):
    """Regularization of a resampled PF's SFV particles (reading F4k): phi += h chol(Sigma) z with
    Sigma = sum_p w_p (phi_p - phi^)(phi_p - phi^)^T / sum w (the posterior belief's second central moment, before
    resampling), h = (4 / ((d + 2) P))^{1/(d + 4)}, d = 3, z ~ N(0, I3) from normals4(key, n, p, 0x700 + 16 s);
    Sigma + 1e-12 tr(Sigma) I, no move when that is not positive definite."""
    if not prm.regularize:
        return phi_res
    P = phi.shape[0]
    d = phi - phi_hat[None, :]
    Sg = (w[:, None] * d).T @ d / np.sum(w)
    Sg = Sg + 1e-12 * np.trace(Sg) * np.eye(3)
    try:
        L = np.linalg.cholesky(Sg)
    except np.linalg.LinAlgError:
        return phi_res
    h = (4.0 / (5.0 * P)) ** (1.0 / 7.0)
    out = phi_res.copy()
    for p in range(P):
        z = O.normals4(prm.key, n, p, ST_PF_REG + 16 * s)[:3]
        out[p] += h * (L @ z)
    return out


def step(base, st: State, y, prm: Params):
    """One time step n = st.n; returns (new State, report dict of the intermediate messages)."""
    n = st.n
    J, Nz = base.J, base.Nz
    y = np.asarray(y).reshape(J, Nz)
    P = st.x.shape[0]
    rep = {}
    # (i) prediction and birth messages
    x, eta, slots = predict(st, prm)
    rep["x_pred"], rep["eta_pred"] = x, eta
    rep["slots_pred"] = [dataclasses.replace(s) for s in slots]
    x_hat = np.mean(x[:, :3], axis=0)                                      # x^_{n|n-1}
    eta_bar = np.mean(eta, axis=1)                                         # eta-bar
    rep["x_pred_hat"], rep["eta_bar"] = x_hat, eta_bar
    next_id = st.next_id
    if len(slots) < S_MAX:
        legacy = [st.phi_hat[s.ident] for s in slots[1:]] if st.phi_hat else []
        b = birth(base, st, prm, x_hat, y, np.array(legacy) if legacy else np.zeros((0, 3)), next_id)
        if b is not None:
            slots.append(b)
            next_id += 1
    rep["n_slots"] = len(slots)
    rep["slots_prior"] = [dataclasses.replace(s) for s in slots]
    S = len(slots)
    orc = _oracle_for(base, S - 1)
    # belief averages of the prediction messages (reading F4c)
    u, m, mw = belief_vectors(orc, x, slots, prm.P_m)
    zeta = np.stack([s.zeta for s in slots], axis=1)                       # [J][S]
    mu3 = zeta[:, :, None] * u                                             # mu~_3 per slot
    mu_nu = np.sum(mu3, axis=1)                                            # sum over S~
    rep["u"], rep["m"], rep["momega"], rep["mu_nu"] = u, m, mw, mu_nu
    # (iii) MT update message iota~ with the moment-matched amplitude priors (C-amb-7) and the paired SFVs (C-amb-8)
    mm = np.zeros((J, S), dtype=complex)
    vv = np.zeros((J, S))
    for s, sl in enumerate(slots):
        eps, mub, gab, _ = stats(sl)
        for j in range(J):
            mm[j, s], vv[j, s] = O.moment_match(mub, gab, eps * sl.zeta[j])
    sfv_pp = np.stack([sl.phi for sl in slots[1:]], axis=1) if S > 1 else np.zeros((P, 0, 3))
    rc, l = orc.loglik(x, sfv_pp.reshape(P, -1), y, mm, vv, eta_bar, sfv_per_particle=True)
    if rc:
        raise ValueError(f"loglik status {rc}")
    rep["l"], rep["prior_m"], rep["prior_v"] = l, mm, vv
    # nu~ with all slots' columns
    rc, _, w_eta, _ = orc.noise_update(eta, np.full((J, P), 1.0 / P), y, mu_nu, m)
    if rc:
        raise ValueError(f"noise status {rc}")
    rep["w_eta"] = w_eta
    # kappa~ and omega~ of every slot with the other slots' terms
    pf_out, ppr_out, w_new = [], [], []
    for s, sl in enumerate(slots):
        others = [t for t in range(S) if t != s]
        mu3o = mu_nu - mu3[:, s]
        mo = m[:, others]
        rc, logr, w, logM, ex = orc.pf_update(x, sl.phi, sl.w, sl.mu, sl.gamma, sl.zeta, eta_bar, y, mu3o, mo)
        if rc:
            raise ValueError(f"pf status {rc}")
        rc, out = orc.ppr_update(sl.zeta, eta_bar, y, mu3o, mo, mw[:, s], u[:, s])
        if rc:
            raise ValueError(f"ppr status {rc}")
        pf_out.append((logr, logM, ex))
        ppr_out.append(out)
        w_new.append(w)
    rep["pf"], rep["ppr"] = pf_out, ppr_out
    # beliefs, estimates, resampling
    rc, x_new, est, lse, anc = O.step_update(l, x, prm.key, n, prm.regularize)
    if rc:
        raise ValueError(f"step_update status {rc}")
    rep["est"], rep["lse"], rep["anc"] = est, lse, anc
    eta_hat = np.sum(w_eta * eta, axis=1)
    eta_new = np.zeros_like(eta)
    for j in range(J):
        rc, a = O.resample(w_eta[j], philox_u32(prm.key, 0, n, ST_NOISE_RES + j)[0])
        eta_new[j] = eta[j, a]
    rep["eta_hat"] = eta_hat
    new_slots, phi_hat, report = [], {}, []
    for s, sl in enumerate(slots):
        w = w_new[s]
        ex = float(np.sum(w))
        zeta_post = ppr_out[s][:, 2].copy()
        post = Slot(sl.phi, sl.mu, sl.gamma, w, zeta_post, sl.ident)
        eps, mub, gab, phib = stats(post)
        report.append(dict(ident=sl.ident, exist=ex, mu=mub, gamma=gab, phi=phib, zeta=zeta_post,
                           declared=ex > prm.T_dec))
        if s > 0 and ex < prm.T_pru:                                       # pruning
            continue
        if ex > 0.0:
            rc, a = O.resample(w, philox_u32(prm.key, 0, n, ST_PF_RES + s)[0])
            phi = None if sl.phi is None else regularize_sfv(sl.phi[a], sl.phi, w, phib, prm, n, s)
            post = Slot(phi, sl.mu[a], sl.gamma[a], np.full(P, ex / P), zeta_post, sl.ident)
        new_slots.append(post)
        if phib is not None:
            phi_hat[sl.ident] = phib
    rep["features"] = report
    new = State(x_new, eta_new, new_slots, n + 1, next_id, phi_hat)
    return new, rep
