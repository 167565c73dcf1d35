"""FMA-pipe rate of the likelihood kernel on shapes where the Horner loop dominates (debug / tuning)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_19723_b200 import cdms, scenes  # noqa: E402

ctx = cdms.Context(0)
for (K, ny, nv, nf, P) in [(6, 2, 4, 8192, 60000), (6, 8, 8, 512, 200000), (4, 8, 8, 128, 400000), (8, 8, 8, 1024, 100000)]:
    cfg = scenes.custom_config("lr", J=1, K=K, ny=ny, nv=nv, nf=nf, P=P, index=3)
    sc = scenes.make_scene(cfg)
    scene = cdms.Scene.from_synthetic(sc)
    x = torch.as_tensor(scenes.make_particles(cfg), device="cuda:0").contiguous()
    dsfv = torch.as_tensor(sc.sfv, device="cuda:0").contiguous()
    y = torch.as_tensor((sc.noise_unit * 0.5).astype(np.complex64), device="cuda:0").contiguous()
    m, v = scenes.priors(sc)
    eta = np.full(cfg.J, 0.02)
    for it in range(2):
        ctx.timing_enable(True)
        cdms.loglik(ctx, scene, x, dsfv, y, m, v, eta)
        ctx.sync()
        ms, n = ctx.timing_read()
    flop = 8.0 * cfg.Nz * P * cfg.J * cfg.S
    print(f"S={cfg.S} Na={cfg.Na} nf={nf} P={P}: K1 {ms:.2f} ms  {flop / ms / 1e9:.1f} TFLOP/s  "
          f"{flop / ms / 1e9 / 74.45 * 100:.1f}% of 74.45")
