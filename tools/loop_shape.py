"""One launch of the likelihood kernel on a loop-dominated shape (S=7, 8 antennas, nf=8192) for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_19723_b200 import cdms, scenes  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ctx = cdms.Context(0)
cfg = scenes.custom_config("ls", J=1, K=6, ny=2, nv=4, nf=nf, P=60000, index=3)
sc = scenes.make_scene(cfg)
scene = cdms.Scene.from_synthetic(sc)
x = torch.as_tensor(scenes.make_particles(cfg), device="cuda:0").contiguous()
dsfv = torch.as_tensor(sc.sfv, device="cuda:0").contiguous()
y = torch.as_tensor((sc.noise_unit * 0.5).astype(np.complex64), device="cuda:0").contiguous()
m, v = scenes.priors(sc)
for it in range(3):
    cdms.loglik(ctx, scene, x, dsfv, y, m, v, np.full(1, 0.02))
ctx.sync()
print("ok")
