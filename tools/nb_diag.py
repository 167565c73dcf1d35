"""GPU diagnostic for the PLANAR_NB tensor-core path: per-component error of c and G against the oracle, for
nb_corr_kernel and for K1 (CDMS_NB_TENSOR=0), and the resulting rel-l.   python tools/nb_diag.py"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as orc  # noqa: E402
from tests.gpu_common import Case, rel_err  # noqa: E402
from tests.helpers import small_cfg  # noqa: E402


def main():
    from paper_2604_19723_b200 import build as B
    B.build()
    from paper_2604_19723_b200 import cdms as cd
    shapes = [dict(J=2, K=3, ny=3, nv=5, nf=100, P=77), dict(J=1, K=4, ny=8, nv=8, nf=128, P=64),
              dict(J=1, K=4, ny=16, nv=16, nf=64, P=60)]
    for shape in shapes:
        cfg = small_cfg(**shape, index=97)
        case = Case(orc, cfg, wavefront="planar_nb", precision="fp32")
        st, co, Go = case.o.terms(case.x, case.sc.sfv, case.y)
        _, lo = case.oracle_loglik()
        for flag in ("1", "0"):
            os.environ["CDMS_NB_TENSOR"] = flag
            ctx = cd.Context(0)
            l, c, G = cd.loglik_terms(ctx, case.scene, case.dx, case.dsfv, case.dy, case.m, case.v, case.eta)
            ctx.sync()
            l, c, G = l.cpu().numpy(), c.cpu().numpy(), G.cpu().numpy()
            ctx.close()
            name = "tensor" if flag == "1" else "K1"
            relc = np.abs(c - co) / np.maximum(np.abs(co), 1e-30)
            ph = np.angle(c * np.conj(co))
            print(f"{shape} {name:6s} |dc|/|c| max per s {np.max(relc, axis=(0, 1))}")
            print(f"{'':>60s} phase err mean per s {np.mean(ph, axis=(0, 1))} max {np.abs(ph).max():.3e}")
            print(f"{'':>60s} |c|/|c_o| - 1 mean {np.mean(np.abs(c) / np.abs(co) - 1):.3e}"
                  f"  G max rel {np.max(np.abs(G - Go)) / cfg.Nz:.3e}"
                  f"  rel-l max {rel_err(l, lo, cfg.J, cfg.Nz).max():.3e}")
    os.environ.pop("CDMS_NB_TENSOR", None)


if __name__ == "__main__":
    main()
