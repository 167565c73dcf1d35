"""Diagnose GPU-vs-oracle log-likelihood gaps: for sampled particles compare
 (1) the oracle, (2) the GPU kernel, (3) the S x S formula evaluated in numpy on the GPU-MATERIALIZED
 responses (cdms_response, same phasor arithmetic as the kernel): (3) - (1) is the phasor error,
 (2) - (3) the Horner / closed-form Gram / fp32 accumulation error.  Also max phase error of psi."""
import argparse
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402
from paper_2604_19723_b200 import scenes  # noqa: E402
from tests.gpu_common import Case, rel_err  # noqa: E402


def ss_loglik(Psi, z, m, v, eta):
    c = Psi.conj().T @ z
    G = Psi.conj().T @ Psi
    e = z - Psi @ m
    M = Psi * np.sqrt(v)[None, :]
    K = np.eye(len(m)) + (M.conj().T @ M) / eta
    b = M.conj().T @ e
    L = np.linalg.cholesky(K)
    x = np.linalg.solve(L, b)
    return (-len(z) * math.log(math.pi * eta) - 2 * np.sum(np.log(np.real(np.diag(L))))
            - np.vdot(e, e).real / eta + np.vdot(x, x).real / eta ** 2), c, G


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--wavefront", default="planar_nb")
    ap.add_argument("--n", type=int, default=24)
    ap.add_argument("--precision", default="fp32")
    a = ap.parse_args()
    from paper_2604_19723_b200 import cdms
    cfg = scenes.CONFIGS[a.config]
    P = min(cfg.P, 4096)
    case = Case(O, cfg, wavefront=a.wavefront, precision=a.precision, P=P)
    ctx = cdms.Context(0)
    lg = case.gpu_loglik(ctx).cpu().numpy()
    ctx.sync()
    idx = scenes.stratified_sample(P, a.n)
    st, lo = case.oracle_loglik(idx)
    rows = []
    for t, i in enumerate(idx):
        p = case.x[i, :3]
        l3 = 0.0
        worst_ph = 0.0
        for j in range(cfg.J):
            js = np.array([(j, s) for s in range(cfg.S)])
            psi_g = cdms.response(ctx, case.scene, np.repeat(p[None], cfg.S, 0), js, case.sc.sfv).cpu().numpy().T
            psi_o = case.o.responses(p, j, case.sc.sfv)
            worst_ph = max(worst_ph, np.max(np.abs(np.angle(psi_g * psi_o.conj()))))
            z = case.y[j].reshape(-1)
            lj, cg, Gg = ss_loglik(psi_g, z, case.m[j], case.v[j], case.eta[j])
            lj_o, co, Go = ss_loglik(psi_o, z, case.m[j], case.v[j], case.eta[j])
            l3 += lj
            dc = np.max(np.abs(cg - co)) / np.linalg.norm(z)
            dG = np.max(np.abs(Gg - Go)) / case.o.Nz
        den = max(abs(lo[t]), cfg.J * cfg.Nz)
        rows.append((i, lo[t], (lg[i] - lo[t]) / den, (l3 - lo[t]) / den, (lg[i] - l3) / den, worst_ph, dc, dG))
    print(f"{a.config} {a.wavefront} {a.precision}: particle, l_orc, rel(gpu-orc), rel(psi_gpu-orc), "
          f"rel(gpu-psi_gpu), max dphase, |dc|/|z| (last j), |dG|/Nz")
    for r in rows:
        print(f"{r[0]:7d} {r[1]:14.4f} {r[2]: .3e} {r[3]: .3e} {r[4]: .3e} {r[5]:.2e} {r[6]:.2e} {r[7]:.2e}")
    e = np.array([abs(r[2]) for r in rows])
    print("max rel gpu-orc", e.max())
    # kernel's own c and G (cdms_loglik_terms) against the oracle's direct sums
    import torch
    sub = torch.as_tensor(case.x[idx], device="cuda:0").contiguous()
    lk, ck, Gk = cdms.loglik_terms(ctx, case.scene, sub, case.dsfv, case.dy, case.m, case.v, case.eta)
    ctx.sync()
    ck, Gk = ck.cpu().numpy(), Gk.cpu().numpy()
    st, co, Go = case.o.terms(case.x[idx], case.sc.sfv, case.y)
    zn = np.array([np.linalg.norm(case.y[j]) for j in range(cfg.J)])
    print("kernel terms: particle, max|dc|/|c| (components with |c| > 0.1 max), max|dc|/(sqrt(Nz)|z|), max|dG|/Nz")
    for t, i in enumerate(idx):
        big = np.abs(co[t]) > 0.1 * np.abs(co[t]).max()
        rc = np.max(np.abs(ck[t] - co[t])[big] / np.abs(co[t])[big])
        rz = np.max(np.abs(ck[t] - co[t]) / (math.sqrt(cfg.Nz) * zn[:, None]))
        rg = np.max(np.abs(Gk[t] - Go[t])) / cfg.Nz
        print(f"{i:7d} {rc:.3e} {rz:.3e} {rg:.3e}")


if __name__ == "__main__":
    main()
