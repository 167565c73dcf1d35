"""Shared set-up for the GPU parity tests: one synthetic scene, consumed by the oracle (fp64 CPU) and by
libcdms (CUDA) on identical inputs.  The measurement y is synthesized with the ORACLE's responses and
rounded once to complex64; both sides then read that complex64 array."""
import numpy as np

from paper_2604_19723_b200 import scenes

# Measured parity maxima, one record per check (written to $PARITY_REPORT by conftest at session end).
REPORT = []
CURRENT = {"test": None}


def record(kind, value, tol, **extra):
    REPORT.append({"test": CURRENT["test"], "kind": kind, "max": float(value), "tol": float(tol), **extra})


class Case:
    def __init__(self, orc, cfg, wavefront="spherical", pathloss=False, precision="fp32", mode="nzm", P=None,
                 particles=None, step=0):
        import torch
        from paper_2604_19723_b200 import cdms
        self.cfg = cfg
        self.sc = scenes.make_scene(cfg, step=step)
        self.o = orc.Oracle.from_scene(self.sc, wavefront=wavefront, pathloss=pathloss)
        y, eta = orc.measurement(self.o, self.sc, scenes.P_TRUE, wavefront=None)
        self.y64 = y.astype(np.complex64)
        self.y = self.y64.astype(np.complex128)     # what both sides consume
        self.eta = np.full(cfg.J, eta)
        self.m, self.v = scenes.priors(self.sc, mode)
        if pathloss:  # path-loss-compensated responses are ~lambda/(4 pi d): rescale the prior
            self.m, self.v = self.m * 0.0, self.v * 1e-4
        P = cfg.P if P is None else P
        self.x = particles if particles is not None else scenes.make_particles(cfg, 0, P)
        self.scene = cdms.Scene.from_synthetic(self.sc, wavefront=wavefront, pathloss=pathloss, precision=precision)
        dev = "cuda:0"
        self.dx = torch.as_tensor(self.x, device=dev).contiguous()
        self.dsfv = torch.as_tensor(self.sc.sfv, device=dev).contiguous()
        self.dy = torch.as_tensor(self.y64, device=dev).contiguous()

    def gpu_loglik(self, ctx, **kw):
        from paper_2604_19723_b200 import cdms
        return cdms.loglik(ctx, self.scene, self.dx, self.dsfv, self.dy, self.m, self.v, self.eta, **kw)

    def oracle_loglik(self, idx=None, **kw):
        x = self.x if idx is None else self.x[idx]
        return self.o.loglik(x, self.sc.sfv, self.y, self.m, self.v, self.eta, **kw)


def rel_err(l_gpu, l_orc, J, Nz):
    """C-amb-11: |l_gpu - l_orc| / max(|l_orc|, J Nz)."""
    den = np.maximum(np.abs(l_orc), J * Nz)
    return np.abs(l_gpu - l_orc) / den
