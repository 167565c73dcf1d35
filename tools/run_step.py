"""Run cdms_bp_step on a BASELINE config for ncu captures / sanitizer runs (no timing, no oracle):
python tools/run_step.py CONFIG [P_local] [--wavefront W] [--precision fp32|fp64] [--steps N]."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_19723_b200 import cdms, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("P", type=int, nargs="?", default=None)
    ap.add_argument("--wavefront", default="spherical")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    cfg = scenes.CONFIGS[a.config]
    P = a.P or cfg.P
    sc = scenes.make_scene(cfg)
    ctx = cdms.Context(0)
    scene = cdms.Scene.from_synthetic(sc, wavefront=a.wavefront, precision=a.precision)
    J, S = cfg.J, cfg.S
    pos = np.repeat(scenes.P_TRUE[None], J * S, axis=0)
    js = np.array([(j, s) for j in range(J) for s in range(S)], dtype=np.int32)
    psi = cdms.response(ctx, scene, pos, js, sc.sfv).reshape(J, S, -1)
    clean = torch.einsum("jsn,s->jn", psi, torch.as_tensor(sc.rho, device="cuda:0"))
    eta = float((clean.abs() ** 2).sum().item()) / (scene.Nz * J) / 100.0
    y = (clean + eta ** 0.5 * torch.as_tensor(sc.noise_unit.reshape(J, -1), device="cuda:0"))
    y = y.to(torch.complex64).reshape(J, cfg.nf, cfg.Na).contiguous()
    m, v = scenes.priors(sc, "nzm")
    x = torch.as_tensor(scenes.make_particles(cfg, 0, P), device="cuda:0").contiguous()
    dsfv = torch.as_tensor(sc.sfv, device="cuda:0").contiguous()
    for n in range(a.steps):
        cdms.bp_step(ctx, scene, x, dsfv, y, m, v, np.full(J, eta), 0.1, 0.5, sc.philox_key, n)
    print("run_step status", ctx.sync(raise_on_error=False), "launches", ctx.launch_count())


if __name__ == "__main__":
    main()
