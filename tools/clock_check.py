"""Sustained-load SM clock during the likelihood kernel: wall time vs clock64 cycles, nvidia-smi sampling."""
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_19723_b200 import cdms, scenes  # noqa: E402

rows = []
proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [rows.append(l.strip()) for l in proc.stdout], daemon=True).start()
ctx = cdms.Context(0)
cfg = scenes.custom_config("lr", J=1, K=6, ny=8, nv=8, nf=512, P=1_000_000, index=3)
sc = scenes.make_scene(cfg)
scene = cdms.Scene.from_synthetic(sc)
x = torch.as_tensor(scenes.make_particles(cfg), device="cuda:0").contiguous()
dsfv = torch.as_tensor(sc.sfv, device="cuda:0").contiguous()
y = torch.as_tensor((sc.noise_unit * 0.5).astype(np.complex64), device="cuda:0").contiguous()
m, v = scenes.priors(sc)
eta = np.full(cfg.J, 0.02)
time.sleep(1.0)
n0 = len(rows)
t0 = time.time()
ctx.timing_enable(True)
for it in range(40):
    cdms.loglik(ctx, scene, x, dsfv, y, m, v, eta)
ctx.sync()
ms, n = ctx.timing_read()
t1 = time.time()
time.sleep(0.5)
proc.terminate()
load = rows[n0 + 2:]
print(f"40 launches, {ms / n:.2f} ms each ({t1 - t0:.1f} s wall); flop rate {8.0 * cfg.Nz * cfg.P * cfg.S / (ms / n) / 1e9:.1f} TFLOP/s")
print("nvidia-smi samples under load (sm MHz, W, reasons):")
for r in load[:: max(1, len(load) // 12)]:
    print("  ", r)
