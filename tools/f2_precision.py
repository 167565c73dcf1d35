"""F2 design check (CPU only): how accurate must the operands of the PLANAR_NB tensor-core contraction be?

PLANAR_NB responses are rank one as an N_f x N_a matrix (oracle/cdms_oracle.c orc_response):
psi[k, m] = B_k A_m.  The tensor path computes W_m = sum_k conj(B_k) y[m, k] as a GEMM and then
c = sum_m conj(A_m) W_m.  This script evaluates c with emulated operand precisions (fp16 hi/lo splits with
fp32 accumulation; subnormal fp16 operands read as zero, as on the tensor core, so both operands are scaled
into fp16's upper range before the split) and reports the
C-amb-11 relative log-likelihood error against the fp64 definition, using the oracle's responses.

    python tools/f2_precision.py [--config c4] [--particles 24]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as orc  # noqa: E402  (design tool, not product code)
from paper_2604_19723_b200 import scenes  # noqa: E402


def loglik_from_terms(c, G, znorm2, m, v, eta, Nz):
    """A5 from c [S] and G [S][S] for one PA, fp64."""
    S = len(c)
    sv = np.sqrt(v)
    K = np.eye(S) + (sv[:, None] * G * sv[None, :]) / eta
    L = np.linalg.cholesky(K)
    g = c - G @ m
    b = sv * g
    e2 = znorm2 - 2 * np.real(np.vdot(m, c)) + np.real(np.vdot(m, G @ m))
    x = np.linalg.solve(L, b)
    return (-Nz * np.log(np.pi * eta) - 2 * np.sum(np.log(np.real(np.diag(L)))) - e2 / eta
            + np.real(np.vdot(x, x)) / eta ** 2)


def ftz16(a):
    """The tensor core reads fp16 subnormals as zero (measured on B200: without operand scaling the lo halves
    of |x| < 1 operands flush and the GPU error matches this model)."""
    return np.where(np.abs(a.astype(np.float32)) < 2.0 ** -14, np.float16(0), a)


def split16(x):
    h = x.astype(np.float16)
    lo = (x - h.astype(np.float32)).astype(np.float16)
    return ftz16(h), ftz16(lo)


A_SCALE = 2.0 ** 14   # |b| <= 1 -> |2^14 b| <= 16384 < 65504; y scaled to max in [2^14, 2^15)


def W_emul(Bc, y, mode):
    """Bc [Nf] complex (unit modulus), y [Na][Nf] complex -> W [Na] = sum_k conj(B_k) y[m,k], fp32 accumulate."""
    br, bi = Bc.real.astype(np.float32), Bc.imag.astype(np.float32)
    yr, yi = y.real.astype(np.float32), y.imag.astype(np.float32)
    scale = 2.0 ** (15 - np.ceil(np.log2(max(np.abs(yr).max(), np.abs(yi).max()))))
    if mode != "fp32":
        br, bi = (br * A_SCALE).astype(np.float32), (bi * A_SCALE).astype(np.float32)
        scale_a = A_SCALE
    else:
        scale_a = 1.0
    yr, yi = (yr * scale).astype(np.float32), (yi * scale).astype(np.float32)
    if mode == "fp32":
        parts = [((br, bi), (yr, yi))]
    else:
        (brh, brl), (bih, bil) = split16(br), split16(bi)
        (yrh, yrl), (yih, yil) = split16(yr), split16(yi)
        f = lambda a: a.astype(np.float32)  # noqa: E731  (products of f16 are exact in f32)
        hh = ((f(brh), f(bih)), (f(yrh), f(yih)))
        hl = ((f(brh), f(bih)), (f(yrl), f(yil)))
        lh = ((f(brl), f(bil)), (f(yrh), f(yih)))
        parts = {"f16x3": [hh, hl, lh], "f16x2_ylo0": [hh, lh], "f16x1": [hh]}[mode]
    # TMEM accumulation: one fp32 add of a K=16 block (8 subcarriers x re/im) per MMA, in issue order
    Wr = np.zeros(y.shape[0], np.float32)
    Wi = np.zeros(y.shape[0], np.float32)
    for k0 in range(0, len(br), 8):
        ks = slice(k0, k0 + 8)
        for (ar, ai), (zr, zi) in parts:
            Wr = (Wr + (zr[:, ks].astype(np.float64) @ ar[ks] + zi[:, ks].astype(np.float64) @ ai[ks])).astype(np.float32)
            Wi = (Wi + (zi[:, ks].astype(np.float64) @ ar[ks] - zr[:, ks].astype(np.float64) @ ai[ks])).astype(np.float32)
    return (Wr.astype(np.float64) + 1j * Wi.astype(np.float64)) / (scale * scale_a)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--particles", type=int, default=24)
    args = ap.parse_args()
    cfg = scenes.CONFIGS[args.config]
    sc = scenes.make_scene(cfg)
    o = orc.Oracle.from_scene(sc, wavefront="planar_nb")
    y, eta = orc.measurement(o, sc, scenes.P_TRUE, wavefront=None)
    y = y.astype(np.complex64).astype(np.complex128)
    m, v = scenes.priors(sc, "nzm")
    x = scenes.make_particles(cfg, 0, args.particles)
    Na, Nf, Nz = cfg.Na, cfg.nf, cfg.Nz
    worst = {}
    for p in range(args.particles):
        for j in range(cfg.J):
            yj = y[j].reshape(Nf, Na).T  # [Na][Nf], element n = k Na + m
            Psi = o.responses(x[p, :3], j, sc.sfv).T  # [S][Nz]
            Psi = Psi.reshape(cfg.S, Nf, Na)
            G = np.conj(Psi.reshape(cfg.S, Nz)) @ Psi.reshape(cfg.S, Nz).T
            c_ex = np.array([np.vdot(Psi[s].reshape(Nz), y[j].reshape(Nz)) for s in range(cfg.S)])
            zn2 = np.real(np.vdot(y[j], y[j]))
            l_ex = loglik_from_terms(c_ex, G, zn2, m[j], v[j], eta, Nz)
            for mode in ("fp32", "f16x3", "f16x2_ylo0", "f16x1"):
                c = np.empty(cfg.S, complex)
                for s in range(cfg.S):
                    Bk = Psi[s][:, 0] / np.abs(Psi[s][:, 0])       # unit-modulus delay factor (x a_0 carrier)
                    Am = Psi[s][0, :] / Psi[s][0, 0] * np.abs(Psi[s][0, 0])
                    Bk32 = (Bk.real.astype(np.float32) + 1j * Bk.imag.astype(np.float32))
                    W = W_emul(Bk32, yj, mode)
                    A32 = (Am.real.astype(np.float32) + 1j * Am.imag.astype(np.float32)).astype(np.complex64)
                    c[s] = np.sum(np.conj(A32).astype(np.complex128) * W.astype(np.complex64))  # fp64 epilogue sum
                l = loglik_from_terms(c, G, zn2, m[j], v[j], eta, Nz)
                e = abs(l - l_ex) / max(abs(l_ex), cfg.J * Nz)
                worst[mode] = max(worst.get(mode, 0.0), e)
    for k, e in worst.items():
        print(f"{args.config} planar_nb {k:12s} max rel_l {e:.3e}")


if __name__ == "__main__":
    main()
