"""ctypes binding of the fp64 CPU oracle (oracle/cdms_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cdms_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

WAVEFRONTS = {"spherical": 0, "planar_wb": 1, "planar_nb": 2}
OK, EINVAL, EDEGENERATE, EZEROMASS = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle: plain fp64, no fast-math, no FMA contraction, OpenMP over particles."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
               "-fPIC", "-shared", "-o", LIB, SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return LIB


class OrcScene(C.Structure):
    _fields_ = [("J", C.c_int32), ("K", C.c_int32), ("ny", C.c_int32), ("nv", C.c_int32),
                ("nf", C.c_int32), ("wavefront", C.c_int32), ("pathloss", C.c_int32),
                ("pad_", C.c_int32), ("dy", C.c_double), ("dv", C.c_double), ("fc", C.c_double),
                ("pa_pos", C.POINTER(C.c_double)), ("pa_rot", C.POINTER(C.c_double)),
                ("f_pb", C.POINTER(C.c_double))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        _lib.orc_philox4x32_10.argtypes = [C.POINTER(C.c_uint32)] * 3
        _lib.orc_step_u_bits.restype = C.c_uint32
        _lib.orc_step_u_bits.argtypes = [C.c_uint64, C.c_uint64]
        _lib.orc_normals4.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, dp]
        _lib.orc_moment_match.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, dp]
        _lib.orc_birth_candidate.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, dp, dp]
        _lib.orc_birth_residual.argtypes = [C.c_void_p, dp, dp, C.c_int, C.c_void_p, C.c_void_p]
        _lib.orc_gamma_draw.restype = C.c_double
        _lib.orc_gamma_draw.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_double]
        _lib.orc_birth_proposal.argtypes = [C.c_void_p, dp, dp, C.c_int, C.c_void_p, dp, C.c_int64, C.c_uint64,
                                            C.c_uint64, dp, dp, dp, dp, C.POINTER(C.c_int64)]
    return _lib


def _d(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


class Oracle:
    """Holds one scene (J PAs, URA, grid) in the oracle's own struct."""

    def __init__(self, pa_pos, pa_rot, ny, nv, dy, dv, f_pb, fc, K, wavefront="spherical",
                 pathloss=False):
        self.pa_pos = _f64(pa_pos).reshape(-1, 3)
        self.pa_rot = _f64(pa_rot).reshape(-1, 3, 3)
        self.f_pb = _f64(f_pb).reshape(-1)
        self.J = self.pa_pos.shape[0]
        self.K = int(K)
        self.S = self.K + 1
        self.ny, self.nv = int(ny), int(nv)
        self.Na = self.ny * self.nv
        self.nf = self.f_pb.shape[0]
        self.Nz = self.Na * self.nf
        self.sc = OrcScene(self.J, self.K, self.ny, self.nv, self.nf, WAVEFRONTS[wavefront],
                           int(bool(pathloss)), 0, float(dy), float(dv), float(fc),
                           _d(self.pa_pos), _d(self.pa_rot), _d(self.f_pb))
        self.wavefront = wavefront

    @classmethod
    def from_scene(cls, scene, wavefront="spherical", pathloss=False):
        cfg = scene.cfg
        return cls(scene.pa_pos, scene.pa_rot, cfg.ny, cfg.nv, scene.dy, scene.dv, cfg.f_pb(),
                   cfg.fc, cfg.K, wavefront=wavefront, pathloss=pathloss)

    # -- geometry -------------------------------------------------------------------------
    def template(self) -> np.ndarray:
        out = np.zeros((3, self.Na))
        lib().orc_template(self.ny, self.nv, C.c_double(self.sc.dy), C.c_double(self.sc.dv), _d(out))
        return out

    def layout(self, sfv):
        sfv = _f64(sfv).reshape(-1, 3)
        assert sfv.shape[0] == self.K
        lay = np.zeros((self.J, self.S, 3, self.Na))
        va = np.zeros((self.J, self.S, 3))
        H = np.zeros((self.S, 3, 3))
        st = lib().orc_layout(C.byref(self.sc), _d(sfv), _d(lay), _d(va), _d(H))
        return st, lay, va, H

    # -- responses ------------------------------------------------------------------------
    def response(self, pos, j, s, sfv, wavefront: Optional[str] = None):
        pos = _f64(pos).reshape(3)
        sfv = _f64(sfv).reshape(-1, 3)
        sv = _f64(sfv[s - 1]) if s > 0 else np.zeros(3)
        out = np.zeros(self.Nz, dtype=np.complex128)
        wf = WAVEFRONTS[wavefront or self.wavefront]
        st = lib().orc_response(C.byref(self.sc), _d(pos), int(j), int(s), _d(sv), wf,
                                out.ctypes.data_as(C.c_void_p))
        return st, out

    def responses(self, pos, j, sfv, wavefront=None) -> np.ndarray:
        """Psi_j(p) in C^{Nz x S} (columns s = 0..K)."""
        cols = []
        for s in range(self.S):
            st, psi = self.response(pos, j, s, sfv, wavefront)
            if st:
                raise ValueError(f"response status {st}")
            cols.append(psi)
        return np.stack(cols, axis=1)

    # -- likelihood ------------------------------------------------------------------------
    def loglik(self, particles, sfv, y, m, v, eta, logw_prior=None, sfv_per_particle=False,
               want_amp=False):
        x = _f64(particles)
        P, pstride = x.shape
        sfv = _f64(sfv)
        y = _c128(y).reshape(self.J, self.nf, self.Na)
        m = _c128(m).reshape(self.J, self.S)
        v = _f64(v).reshape(self.J, self.S)
        eta = _f64(eta).reshape(self.J)
        lw = None if logw_prior is None else _f64(logw_prior)
        out = np.zeros(P)
        amp = np.zeros((P, self.J, self.S), dtype=np.complex128) if want_amp else None
        st = lib().orc_loglik(C.byref(self.sc), _d(x), C.c_int64(P), C.c_int(pstride), _d(sfv),
                              int(bool(sfv_per_particle)), y.ctypes.data_as(C.c_void_p),
                              m.ctypes.data_as(C.c_void_p), _d(v), _d(eta),
                              _d(lw) if lw is not None else None, _d(out),
                              amp.ctypes.data_as(C.c_void_p) if amp is not None else None)
        return (st, out, amp) if want_amp else (st, out)

    def terms(self, particles, sfv, y, sfv_per_particle=False):
        """(c [P][J][S], G [P][J][S][S]) by direct sums over the element-wise responses."""
        x = _f64(particles)
        P, pstride = x.shape
        y = _c128(y).reshape(self.J, self.nf, self.Na)
        c = np.zeros((P, self.J, self.S), dtype=np.complex128)
        G = np.zeros((P, self.J, self.S, self.S), dtype=np.complex128)
        st = lib().orc_terms(C.byref(self.sc), _d(x), C.c_int64(P), C.c_int(pstride), _d(_f64(sfv)),
                             int(bool(sfv_per_particle)), y.ctypes.data_as(C.c_void_p),
                             c.ctypes.data_as(C.c_void_p), G.ctypes.data_as(C.c_void_p))
        return st, c, G

    # -- F3 birth proposal ---------------------------------------------------
    def birth_residual(self, x_hat, sfv_legacy, y):
        """z~_j = (I - Psi_j Psi_j^dagger) z_j for all PAs, [J][Nz] complex128."""
        sl = _f64(np.asarray(sfv_legacy, dtype=np.float64).reshape(-1, 3))
        y = _c128(y).reshape(self.J, self.Nz)
        out = np.zeros((self.J, self.Nz), dtype=np.complex128)
        st = lib().orc_birth_residual(C.cast(C.byref(self.sc), C.c_void_p), _d(_f64(x_hat)), _d(sl),
                                      int(sl.shape[0]), y.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p))
        return st, out

    def birth_proposal(self, x_hat, sfv_legacy, y, box, N_g, key, counter):
        """(status, P_B [N_g], candidates [N_g][3], mu [3], C [3][3], i*) of the coherent Bartlett proposal."""
        sl = _f64(np.asarray(sfv_legacy, dtype=np.float64).reshape(-1, 3))
        y = _c128(y).reshape(self.J, self.Nz)
        pb = np.zeros(N_g)
        cand = np.zeros((N_g, 3))
        mu = np.zeros(3)
        cov = np.zeros(9)
        ist = C.c_int64(-1)
        st = lib().orc_birth_proposal(C.cast(C.byref(self.sc), C.c_void_p), _d(_f64(x_hat)), _d(sl),
                                      int(sl.shape[0]), y.ctypes.data_as(C.c_void_p), _d(_f64(box)),
                                      C.c_int64(N_g), C.c_uint64(key), C.c_uint64(counter), _d(pb), _d(cand),
                                      _d(mu), _d(cov), C.byref(ist))
        return st, pb, cand, mu, cov.reshape(3, 3), int(ist.value)

    def pf_update(self, particles, phi, walpha, mu, gamma, zeta, eta, y, mu3, mcols):
        """F1: (status, logr [P], w [P], log M_y, existence) of the PF update message kappa~ at the paired PF particles
        (orc_pf_update).  y, mu3: [J][Nz]; mcols: [J][L][Nz]; phi None for the LOS PF."""
        x = _f64(particles)
        P, pstride = x.shape
        phi = None if phi is None else _f64(phi).reshape(P, 3)   # None: the LOS PF s = 0
        mc = _c128(mcols).reshape(self.J, -1, self.Nz)
        L = mc.shape[1]
        y = _c128(y).reshape(self.J, self.Nz)
        mu3 = _c128(mu3).reshape(self.J, self.Nz)
        mu = _c128(mu).reshape(P)
        logr, w, out = np.zeros(P), np.zeros(P), np.zeros(2)
        st = lib().orc_pf_update(C.byref(self.sc), _d(x), C.c_int64(P), C.c_int(pstride),
                                 None if phi is None else _d(phi),
                                 _d(_f64(walpha)), mu.ctypes.data_as(C.c_void_p), _d(_f64(gamma)),
                                 _d(_f64(zeta)), _d(_f64(eta)), y.ctypes.data_as(C.c_void_p),
                                 mu3.ctypes.data_as(C.c_void_p), mc.ctypes.data_as(C.c_void_p), C.c_int(L),
                                 _d(logr), _d(w), _d(out))
        return st, logr, w, float(out[0]), float(out[1])

    def noise_update(self, eta, wxi, y, mu, mcols):
        """nu~ at the noise particles (orc_noise_update): (status, logw [J][P], w [J][P], lognorm [J])."""
        eta = _f64(eta).reshape(self.J, -1)
        P = eta.shape[1]
        wxi = _f64(wxi).reshape(self.J, P)
        mc = _c128(mcols).reshape(self.J, -1, self.Nz)
        S = mc.shape[1]
        y = _c128(y).reshape(self.J, self.Nz)
        mu = _c128(mu).reshape(self.J, self.Nz)
        logw, w, ln = np.zeros((self.J, P)), np.zeros((self.J, P)), np.zeros(self.J)
        st = lib().orc_noise_update(C.byref(self.sc), _d(eta), _d(wxi), C.c_int64(P), y.ctypes.data_as(C.c_void_p),
                                    mu.ctypes.data_as(C.c_void_p), mc.ctypes.data_as(C.c_void_p), C.c_int(S),
                                    _d(logw), _d(w), _d(ln))
        return st, logw, w, ln

    def ppr_update(self, zeta, eta, y, mu3, mcols, momega, mu4):
        """omega~ and the PPR existence (orc_ppr_update): (status, out [J][3] = (log ratio, u, sigma(u)))."""
        mc = _c128(mcols).reshape(self.J, -1, self.Nz)
        L = mc.shape[1]
        out = np.zeros((self.J, 3))
        st = lib().orc_ppr_update(C.byref(self.sc), _d(_f64(zeta)), _d(_f64(eta)),
                                  _c128(y).reshape(self.J, self.Nz).ctypes.data_as(C.c_void_p),
                                  _c128(mu3).reshape(self.J, self.Nz).ctypes.data_as(C.c_void_p),
                                  mc.ctypes.data_as(C.c_void_p), C.c_int(L),
                                  _c128(momega).reshape(self.J, self.Nz).ctypes.data_as(C.c_void_p),
                                  _c128(mu4).reshape(self.J, self.Nz).ctypes.data_as(C.c_void_p), _d(out))
        return st, out

    def bp_step(self, particles, sfv, y, m, v, eta, T, sigma_v, key, step, regularize=True):
        x = _f64(particles).copy()
        P = x.shape[0]
        y = _c128(y).reshape(self.J, self.nf, self.Na)
        m = _c128(m).reshape(self.J, self.S)
        v = _f64(v).reshape(self.J, self.S)
        eta = _f64(eta).reshape(self.J)
        est = np.zeros(28)
        lse = np.zeros(1)
        anc = np.zeros(P, dtype=np.int64)
        st = lib().orc_bp_step(C.byref(self.sc), _d(x), C.c_int64(P), _d(_f64(sfv)),
                               y.ctypes.data_as(C.c_void_p), m.ctypes.data_as(C.c_void_p), _d(v),
                               _d(eta), C.c_double(T), C.c_double(sigma_v), C.c_uint64(key),
                               C.c_uint64(step), int(bool(regularize)), _d(est), _d(lse),
                               anc.ctypes.data_as(C.c_void_p))
        return st, x, est, float(lse[0]), anc


# -- scene-free entry points -------------------------------------------------------------------
def normalize(loglik):
    l = _f64(loglik)
    w = np.zeros_like(l)
    lse = np.zeros(1)
    st = lib().orc_normalize(_d(l), C.c_int64(l.shape[0]), _d(w), _d(lse))
    return st, w, float(lse[0])


def moments(x, w):
    x = _f64(x)
    w = _f64(w)
    est = np.zeros(28)
    st = lib().orc_moments(_d(x), _d(w), C.c_int64(w.shape[0]), _d(est))
    return st, est


def resample(w, u_bits):
    w = _f64(w)
    anc = np.zeros(w.shape[0], dtype=np.int64)
    st = lib().orc_resample(_d(w), C.c_int64(w.shape[0]), C.c_uint32(u_bits),
                            anc.ctypes.data_as(C.c_void_p))
    return st, anc


def resample_loglik(l, u_bits):
    """Systematic resampling of the masses e^{l - max l} (the BP step's quantization, C-amb-23)."""
    l = _f64(l)
    anc = np.zeros(l.shape[0], dtype=np.int64)
    st = lib().orc_resample_loglik(_d(l), C.c_int64(l.shape[0]), C.c_uint32(u_bits), anc.ctypes.data_as(C.c_void_p))
    return st, anc


def step_update(l, particles, key, step, regularize=True):
    """The belief update after the likelihood (normalize, moments, resample, gather, regularize):
    (status, particles out, est [28], lse, ancestors)."""
    l = _f64(l)
    x = _f64(particles).copy()
    P = x.shape[0]
    est = np.zeros(28)
    lse = np.zeros(1)
    anc = np.zeros(P, dtype=np.int64)
    st = lib().orc_step_update(_d(l), _d(x), C.c_int64(P), C.c_uint64(key), C.c_uint64(step), int(bool(regularize)),
                               _d(est), _d(lse), anc.ctypes.data_as(C.c_void_p))
    return st, x, est, float(lse[0]), anc


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (C.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (C.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return [int(x) for x in o]


def normals4(key, step, index, stream):
    out = np.zeros(4)
    lib().orc_normals4(C.c_uint64(key), C.c_uint64(step), C.c_uint64(index), C.c_uint32(stream), _d(out))
    return out


def gamma_draw(key, step, index, stream, c) -> float:
    """One Gamma(c, 1) draw (orc_gamma_draw: Marsaglia-Tsang on Philox blocks (index, step, stream + attempt))."""
    return float(lib().orc_gamma_draw(C.c_uint64(key), C.c_uint64(step), C.c_uint64(index), C.c_uint32(stream),
                                      C.c_double(c)))


def step_u_bits(key, step) -> int:
    return int(lib().orc_step_u_bits(C.c_uint64(key), C.c_uint64(step)))


def predict(x, p0, T, sigma_v, key, step):
    x = _f64(x).copy()
    lib().orc_predict(_d(x), C.c_int64(x.shape[0]), C.c_int64(p0), C.c_double(T), C.c_double(sigma_v),
                      C.c_uint64(key), C.c_uint64(step))
    return x


def regularize(x, p0, P_total, cov21, key, step):
    x = _f64(x).copy()
    cov = _f64(cov21)
    lib().orc_regularize(_d(x), C.c_int64(x.shape[0]), C.c_int64(p0), C.c_int64(P_total), _d(cov),
                         C.c_uint64(key), C.c_uint64(step))
    return x


def birth_candidate(key, counter, i, box):
    out = np.zeros(3)
    lib().orc_birth_candidate(C.c_uint64(key), C.c_uint64(counter), C.c_int64(i), _d(_f64(box)), _d(out))
    return out


def moment_match(mu, gamma, exist):
    out = np.zeros(3)
    lib().orc_moment_match(float(np.real(mu)), float(np.imag(mu)), float(gamma), float(exist), _d(out))
    return complex(out[0], out[1]), float(out[2])


def measurement(orc: Oracle, scene, p_true, wavefront=None, snr=100.0):
    """Synthetic z^(j) = sum_s rho_s psi_s(p_true) + sqrt(eta) w with eta set by
    SNR = P_ch/eta, P_ch = 1/(Nz J) sum_j ||sum_s rho_s psi_s||^2.  Built with the
    oracle's responses; returns (y [J][nf][Na] complex128, eta)."""
    J = orc.J
    clean = np.zeros((J, orc.Nz), dtype=np.complex128)
    for j in range(J):
        Psi = orc.responses(p_true, j, scene.sfv, wavefront)
        clean[j] = Psi @ scene.rho
    pch = float(np.sum(np.abs(clean) ** 2)) / (orc.Nz * J)
    eta = pch / snr
    y = clean + np.sqrt(eta) * scene.noise_unit.reshape(J, orc.Nz)
    return y.reshape(J, orc.nf, orc.Na), eta
