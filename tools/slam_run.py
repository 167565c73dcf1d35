"""F4 demonstration: the SLAM step driver (cdms_slam_step) over an Experiment-1-shaped synthetic track.

Scene: the `exp1` config (J = 4 PAs with 4 x 4 URAs, N_f = 10 over 100 MHz at 3.5 GHz, K = 4 walls) with
the synthetic room of scenes.py; the MT moves from P_TRUE with the constant velocity V_TRUE; each step's snapshot is
z_n^(j) = sum_s rho_s psi_s(p_n) + sqrt(eta) w_n (libcdms responses, fresh CN(0, 1) noise per step, SNR 20 dB at n = 1,
P:L3823-3829).  The method's constants are Experiment 1's; what differs from the paper's setup
(DESIGN.md section 8e): the MT particles start around the true initial state (N(p_0, 0.1^2 I), velocities
N(v_0, 0.1^2 I)) instead of uniformly over the ROI, the noise particles log-uniformly over [0.1, 10] x the true eta
(the paper's [1e-9, 1e-4] assumes its path-loss scale), and the SFV birth box covers this room's walls.

Prints one JSON line per step (position error, declared PFs, SFV errors) and a summary line.  Needs a GPU."""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_19723_b200 import scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="exp1", choices=sorted(scenes.CONFIGS))
    ap.add_argument("--particles", type=int, default=100_000)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--P-m", type=int, default=256)
    ap.add_argument("--N-g", type=int, default=1 << 14)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--init", default="scratch", choices=["scratch", "map", "roi"],
                    help="scratch: the LOS alone (P:L3676), MT particles around the true start; map: LOS + every wall "
                         "as PFs with 5 cm SFV and 10%% amplitude errors (tracking with a rough prior map); roi: the LOS "
                         "alone and MT positions uniform over the ROI (the paper's f(x_0), P:L3673), velocities "
                         "N(0, 0.5^2 I)")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    from paper_2604_19723_b200 import build as B
    B.build()
    from paper_2604_19723_b200 import cdms as cd
    dev = "cuda:0"
    cfg = scenes.CONFIGS[args.config]
    sc = scenes.make_scene(cfg)
    scene = cd.Scene.from_synthetic(sc, precision=args.precision)
    ctx = cd.Context(0)
    J, S, P = cfg.J, cfg.S, args.particles
    T = 0.1
    truth = [scenes.P_TRUE + scenes.V_TRUE * T * n for n in range(args.steps + 1)]
    js = np.array([(j, s) for j in range(J) for s in range(S)], dtype=np.int32)
    rho = torch.as_tensor(sc.rho, device=dev)
    gen = torch.Generator(device=dev).manual_seed(cfg.seed)

    def snapshot(p, eta=None):
        psi = cd.response(ctx, scene, np.repeat(p[None], J * S, axis=0), js, sc.sfv).reshape(J, S, -1)
        clean = torch.einsum("jsn,s->jn", psi, rho)
        if eta is None:
            eta = float((clean.abs() ** 2).sum().item()) / (scene.Nz * J) / 100.0
        w = torch.complex(torch.randn(clean.shape, generator=gen, device=dev, dtype=torch.float64),
                          torch.randn(clean.shape, generator=gen, device=dev, dtype=torch.float64)) / math.sqrt(2.0)
        y = (clean + math.sqrt(eta) * w).to(torch.complex64).reshape(J, scene.nf, scene.Na).contiguous()
        return y, eta

    _, eta_true = snapshot(truth[1])
    box = (-10.0, -5.0, -4.0, 12.0, 12.0, 6.0)
    slam = cd.Slam(ctx, scene, P, T=T, P_m=args.P_m, N_g=args.N_g, box=box)
    rng = np.random.default_rng(cfg.seed)
    walls_sfv = sc.sfv
    x0 = np.zeros((P, 6))
    if args.init == "roi":
        x0[:, :3] = scenes.ROI_LO + (scenes.ROI_HI - scenes.ROI_LO) * rng.uniform(size=(P, 3))
        x0[:, 3:] = 0.5 * rng.standard_normal((P, 3))
    else:
        x0[:, :3] = truth[0] + 0.1 * rng.standard_normal((P, 3))
        x0[:, 3:] = scenes.V_TRUE + 0.1 * rng.standard_normal((P, 3))
    eta0 = eta_true * 10.0 ** rng.uniform(-1.0, 1.0, (J, P))
    slam.init(torch.as_tensor(x0, device=dev), torch.as_tensor(eta0, device=dev))
    if args.init == "map":   # a rough prior map: slots 1..K at the true walls (tracking-mode demonstration)
        v = slam.view()
        amp = sc.rho * (1.0 + 0.1 * (rng.standard_normal(S) + 1j * rng.standard_normal(S)) / math.sqrt(2.0))
        for s_ in range(S):
            if s_:
                v["phi"][s_].copy_(torch.as_tensor(walls_sfv[s_ - 1][None, :] + 0.05 * rng.standard_normal((P, 3))))
            v["mu"][s_].fill_(complex(amp[s_]))
            v["gamma"][s_].fill_(0.01)
            v["w"][s_].fill_(0.9 / P)
        slam.set_slots(list(range(S)), np.full((S, J), 0.9), np.vstack([np.zeros(3), walls_sfv]), n=1, next_id=S)
    walls = sc.sfv
    rows, t_step = [], []
    for n in range(1, args.steps + 1):
        y, _ = snapshot(truth[n], eta_true)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = slam.step(y)
        t_step.append(time.perf_counter() - t0)
        err = float(np.linalg.norm(r["est"][1:4] - truth[n]))
        feats = []
        for i in range(r["n_feat"]):
            if r["ident"][i] == 0 or not r["declared"][i]:
                continue
            d = np.linalg.norm(walls - r["phi_hat"][i][None, :], axis=1)
            feats.append(dict(ident=r["ident"][i], exist=round(float(r["exist"][i]), 4),
                              phi=[round(float(v), 3) for v in r["phi_hat"][i]], nearest_wall=int(np.argmin(d)),
                              sfv_err=round(float(d.min()), 4)))
        row = dict(n=n, pos_err_m=round(err, 5), los_exist=round(float(r["exist"][0]), 4),
                   n_slots=r["n_slots"], declared=feats,
                   eta_ratio=[round(float(v / eta_true), 3) for v in r["eta_hat"]], step_ms=round(1e3 * t_step[-1], 2))
        rows.append(row)
        print(json.dumps(row), flush=True)
    errs = np.array([r["pos_err_m"] for r in rows])
    tail = errs[len(errs) // 2:]
    summary = dict(summary=True, config=args.config, init=args.init, particles=P, steps=args.steps,
                   precision=args.precision,
                   pos_err_rmse_second_half_m=float(np.sqrt(np.mean(tail ** 2))), pos_err_final_m=float(errs[-1]),
                   declared_final=len(rows[-1]["declared"]),
                   walls_found=sorted({f["nearest_wall"] for f in rows[-1]["declared"] if f["sfv_err"] < 0.2}),
                   step_ms_median=float(np.median(t_step) * 1e3), wavelength_m=cfg.lam)
    print(json.dumps(summary), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
            f.write(json.dumps(summary) + "\n")
    slam.close()
    ctx.close()


if __name__ == "__main__":
    main()
