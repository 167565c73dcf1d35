"""Per-phase cycle attribution of the likelihood kernel K1 (debug build libcdms_timing.so, -DCDMS_PHASE_TIMING).
Phases: 0 per-(s,p) setup+barrier, 1 NB Gram, 2 per-(s,m) setup, 3 Horner (incl. TMA waits), 4 barrier after
Horner, 5 c-accum + Gram, 6 barrier after Gram, 7 hand-off + barrier."""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CDMS_LIB"] = os.path.join(ROOT, "paper_2604_19723_b200", "libcdms_timing.so")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_19723_b200 import cdms, scenes  # noqa: E402

NAMES = ["setup_ps", "nb_gram", "setup_sm", "horner", "bar_pub", "gram+cacc", "bar_gram", "handoff"]
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--particles", type=int, default=200_000)
ap.add_argument("--wavefront", default="spherical")
a = ap.parse_args()
cfg = scenes.CONFIGS[a.config]
sc = scenes.make_scene(cfg)
scene = cdms.Scene.from_synthetic(sc, wavefront=a.wavefront)
ctx = cdms.Context(0)
P = min(a.particles, cfg.P)
x = torch.as_tensor(scenes.make_particles(cfg, 0, P), device="cuda:0").contiguous()
dsfv = torch.as_tensor(sc.sfv, device="cuda:0").contiguous()
y = torch.as_tensor((sc.noise_unit * 0.5).astype(np.complex64), device="cuda:0").contiguous()
m, v = scenes.priors(sc)
eta = np.full(cfg.J, 0.02)
L = cdms.lib()
L.cdms_debug_phase_read.argtypes = [C.POINTER(C.c_double), C.c_int]
buf = (C.c_double * 8)()
cdms.loglik(ctx, scene, x, dsfv, y, m, v, eta)
ctx.sync()
L.cdms_debug_phase_read(buf, 1)
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record()
cdms.loglik(ctx, scene, x, dsfv, y, m, v, eta)
t1.record()
ctx.sync()
L.cdms_debug_phase_read(buf, 1)
tot = sum(buf)
print(f"{a.config} {a.wavefront} P={P}: loglik {t0.elapsed_time(t1):.2f} ms; per-warp cycle shares:")
for n, b in zip(NAMES, buf):
    print(f"  {n:10s} {b / tot * 100:6.2f}%")
