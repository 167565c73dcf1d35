"""Benchmark of the coherent-likelihood BP step (BASELINE.json metric: particle x VA coherent likelihood
evals/s and ms per BP step at 1/2/4/8 B200).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--particles P_total] [--impl cdms|reference]

One process per GPU (`--gpus N` launches torch.distributed.run itself when WORLD_SIZE is unset).  A step = one
cdms_bp_step (predict, coherent log-likelihood over all particles x PAs x components, LSE normalization, moments,
systematic resampling with redistribution, regularization).  Strong scaling (SURVEY 8(d) metric 2): the default is
c5 (J=4, S=9, 8x8 URA, nf=1024) with P_total = 16M particles split over the N GPUs (P_local = 16M/N).  Inputs are
synthetic (scenes.py recipe); the measurement y is synthesized on the device with libcdms's own responses.
L2 is flushed (256 MiB write) between timed steps; each step is timed with CUDA events on the context's
stream; the reported time is the max over ranks.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2604_19723_b200 import scenes  # noqa: E402

METRIC = "particle x VA coherent likelihood evals/s (BP step)"
UNIT = "evals/s"
FFMA_PER_SM_CLK = 128          # FP32 lanes per SM (cc 10.0), measured 123-128 in tools/microbench
N_SM = 148


def fp32_peak_tflops(mhz: float) -> float:
    return 2.0 * FFMA_PER_SM_CLK * N_SM * mhz * 1e6 / 1e12


def measured_tensor_peak():
    """(dense bf16 TFLOP/s sustained, basis) from the driver-written MEASURED_PEAKS.json; fp16 has the same nominal
    dense rate as bf16 on sm_100 (B200_PROFILING.md), so the bf16 figure is the kind::f16 peak."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["bf16_tflops_sustained"]), "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS 8192^3, 4 s)"
    except (OSError, KeyError, ValueError):
        return 2250.0 * 0.72, "fallback: nominal 2.25 PFLOP/s x 0.72"


def taylor_path(args) -> bool:
    """Spherical / planar WB in fp32 evaluate the correlation with K1T (taylor.cu) unless CDMS_TAYLOR=0."""
    return (args.wavefront != "planar_nb" and args.precision == "fp32"
            and os.environ.get("CDMS_TAYLOR", "1") != "0")


def nb_tensor_path(args) -> bool:
    """PLANAR_NB in fp32 runs the likelihood on the tensor cores (nbmma.cu) unless CDMS_NB_TENSOR=0."""
    return (args.wavefront == "planar_nb" and args.precision == "fp32"
            and os.environ.get("CDMS_NB_TENSOR", "1") != "0")


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML polled every ~2 ms by a thread
    (short timed regions still get samples), nvidia-smi -lms 100 as the fallback when NVML is unavailable."""

    NVML_BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        self.index = int(ids[index]) if index < len(ids) and ids[index].isdigit() else index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def _sample_nvml(self, nv, h) -> bool:
        try:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        except Exception:
            return False
        self.rows.append([str(sm), str(mx), ""] +
                         ["Active" if rs & self.NVML_BITS[k] else "Not Active"
                          for k in ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")])
        return True

    def mark(self):
        """One synchronous sample (call while the timed work is still queued on the GPU)."""
        if self.nvml is not None:
            self._sample_nvml(self.nvml, self.h)

    def _poll_nvml(self, nv, h):
        while not self.stop.is_set() and self._sample_nvml(nv, h):
            self.stop.wait(0.002)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = nv
            self.h = h
            self.t = threading.Thread(target=self._poll_nvml, args=(nv, h), daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.nvml is not None:
            self.stop.set()
            self.t.join(timeout=1)
            return
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def self_launch(args) -> int:
    """`--gpus N` without a torchrun environment: re-run this command under torch.distributed.run with N ranks on
    this node (rendezvous on 127.0.0.1) and relay its output."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def synth_measurement(cd, ctx, scene, sc, torch, dev):
    """z^(j) = sum_s rho_s psi_s(p_true) + sqrt(eta) w with libcdms's responses; SNR 20 dB."""
    J, S = sc.cfg.J, sc.cfg.S
    pos = np.repeat(scenes.P_TRUE[None], J * S, axis=0)
    js = np.array([(j, s) for j in range(J) for s in range(S)], dtype=np.int32)
    psi = cd.response(ctx, scene, pos, js, sc.sfv).reshape(J, S, -1)
    rho = torch.as_tensor(sc.rho, device=dev)
    clean = torch.einsum("jsn,s->jn", psi, rho)
    pch = float((clean.abs() ** 2).sum().item()) / (scene.Nz * J)
    eta = pch / 100.0
    noise = torch.as_tensor(sc.noise_unit.reshape(J, -1), device=dev)
    y = (clean + math.sqrt(eta) * noise).to(torch.complex64).reshape(J, scene.nf, scene.Na).contiguous()
    return y, np.full(J, eta)


def p_total_of(args, cfg) -> int:
    return cfg.P if args.particles is None else args.particles


def run_cdms(args):
    """Strong scaling (SURVEY 8(d) metric 2): P_total particles of the config split over the ranks, P_local each."""
    import torch
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_2604_19723_b200 import build as B
    if rank == 0 and not os.path.exists(os.path.join(ROOT, "paper_2604_19723_b200", "libcdms.so")):
        B.build()
    if world > 1:
        torch.distributed.barrier()
    from paper_2604_19723_b200 import cdms

    dev = f"cuda:{local}"
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream(local)
    cfg = scenes.CONFIGS[args.config]
    P_total = p_total_of(args, cfg)
    if P_total % world:
        raise SystemExit(f"P_total={P_total} is not divisible by {world} ranks")
    P_local = P_total // world
    sc = scenes.make_scene(cfg)
    scene = cdms.Scene.from_synthetic(sc, wavefront=args.wavefront, precision=args.precision)
    ctx = cdms.Context(local, stream)
    if world > 1:
        ctx.comm_init_from_torch(rank, world)
    y, eta = synth_measurement(cdms, ctx, scene, sc, torch, dev)
    m, v = scenes.priors(sc, "nzm")
    x = torch.as_tensor(scenes.make_particles(cfg, rank * P_local, P_local), device=dev).contiguous()
    dsfv = torch.as_tensor(sc.sfv, device=dev).contiguous()
    est = torch.empty(28, dtype=torch.float64, device=dev)
    lse = torch.empty(1, dtype=torch.float64, device=dev)
    ctx.reserve(scene, P_local)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    T, sv, key = 0.1, 0.5, sc.philox_key

    def step(n):
        cdms.bp_step(ctx, scene, x, dsfv, y, m, v, eta, T, sv, key, n, regularize=True, est=est, lse=lse)

    def barrier():
        torch.cuda.synchronize(local)
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize(local)

    for n in range(args.warmup):
        step(n)
    ctx.sync()
    barrier()

    # ---- timed region (device-resident inputs)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    ctx.timing_enable(True)
    with ClockSampler(local) as clk:
        barrier()
        for n in range(args.steps):
            flush.zero_()                       # L2 flush between timed steps (outside the events)
            ev[n][0].record(stream)
            step(args.warmup + n)
            ev[n][1].record(stream)
            if n == args.steps // 2:
                clk.mark()
        clk.mark()
        barrier()
    st = ctx.sync(raise_on_error=False)
    gpu_launches = ctx.launch_count() - launches0
    stage_ms, k_n = ctx.timing_read_stages()      # [correlation, Gram, assembly] summed over the timed steps
    ctx.timing_enable(False)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot = torch.tensor([sum(step_ms)] + stage_ms, dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.MAX)
    ms_per_step = tot[0].item() / args.steps
    n_batches = max(k_n, 1)
    kern_ms = {"corr": tot[1].item() / n_batches, "gram": tot[2].item() / n_batches, "asm": tot[3].item() / n_batches}
    launches_per_step = n_batches / args.steps      # > 1 when the terms budget batches the particles

    # ---- end to end: host measurement in, host estimate out, through the public API
    y_host = torch.empty(y.shape, dtype=torch.complex64, pin_memory=True)
    y_host.copy_(y.cpu())
    est_host = torch.empty(29, dtype=torch.float64, pin_memory=True)
    y_dev = torch.empty_like(y)
    out_dev = torch.empty(29, dtype=torch.float64, device=dev)
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    for n in range(args.steps):
        flush.zero_()
        e2e_ev[n][0].record(stream)
        y_dev.copy_(y_host, non_blocking=True)
        cdms.bp_step(ctx, scene, x, dsfv, y_dev, m, v, eta, T, sv, key, 10_000 + n, est=out_dev[:28], lse=out_dev[28:])
        est_host.copy_(out_dev, non_blocking=True)
        e2e_ev[n][1].record(stream)
    barrier()
    e2e_local = sum(a.elapsed_time(b) for a, b in e2e_ev)
    e2e_t = torch.tensor([e2e_local], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(e2e_t, op=torch.distributed.ReduceOp.MAX)
    e2e_ms = e2e_t.item() / args.steps
    ctx.sync(raise_on_error=False)

    evals_step = P_total * cfg.J * cfg.S
    value = evals_step / (ms_per_step / 1e3)
    result = None
    if rank == 0:
        clocks = clk.summary()
        roof = roofline(args, cfg, P_local, kern_ms, launches_per_step, ms_per_step, clocks)
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64", "data": "synthetic",
            "config": config_dict(args, cfg, P_total, world),
            "roofline": roof,
            "kernel_ms_per_step": {k: round(v * launches_per_step, 4) for k, v in kern_ms.items()},
            "e2e": {"value": evals_step / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(y.numel() * 8), "d2h_bytes_per_step": 29 * 8},
            "clocks": clocks, "gpu_launches": int(gpu_launches), "sync_status": st,
        }
    ctx.close()
    del x, flush
    torch.cuda.empty_cache()
    if rank == 0 and world == 1:
        if not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline(args, cfg, sc, budget_s=args.cpu_seconds)
        if not args.no_extras:
            # C-amb-18(ii): FP32 end-to-end weight error against the oracle (every particle of c2), and the FP64
            # mode's throughput (the mode that meets the 1e-5 weight tolerance end to end)
            result["fp32_weights_vs_oracle"] = fp32_weight_error(cdms, torch, dev)
            result["fp64_mode"] = fp64_mode_line(cdms, torch, dev, local)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return result


def roofline(args, cfg, P_local, kern_ms, launches_per_step, ms_per_step, clocks):
    """The dominant likelihood kernel against its pipe: achieved = its own FMA-pipe / XU
    thread-instructions per launch (committed ncu capture of this config, profiles/pipe_inst.json, per particle x
    P_local) over its live CUDA-event time; peak = 128 FMA lanes (16 XU lanes) x 148 SMs x 1965 MHz.  The direct
    correlation's flop count (8 N_z per (particle, PA, component)) is reported separately as
    direct_equiv_frac: the K1T engine does not execute those flops."""
    dom = max(("corr", "gram"), key=lambda k: kern_ms[k])
    t = kern_ms[dom] / 1e3
    mhz = 1965.0
    peak_fma = 128 * N_SM * mhz * 1e6 / 1e12      # T thread-instructions / s
    peak_xu = 16 * N_SM * mhz * 1e6 / 1e12
    names = kernel_names(args, cfg, P_local)
    flop_launch = 8.0 * cfg.Nz * P_local * cfg.J * cfg.S / launches_per_step
    direct = flop_launch / ((kern_ms["corr"] + kern_ms["gram"]) / 1e3) / 1e12
    roof = {"bound": "alu", "pipe": "fp32 FMA pipe (own instructions)", "kernel": names[dom],
            "kernel_ms": round(kern_ms[dom], 4),
            "kernel_share_of_step": round(kern_ms[dom] * launches_per_step / ms_per_step, 4),
            "launches_per_step": launches_per_step, "unit": "T thread-inst/s",
            "peak": round(peak_fma, 3), "peak_basis": "128 FFMA lanes/SM/clk x 148 SM x 1965 MHz (sm_max); XU: 16",
            "other_kernel": {"name": names["gram" if dom == "corr" else "corr"],
                             "kernel_ms": round(kern_ms["gram" if dom == "corr" else "corr"], 4)},
            "direct_equiv_frac": round(direct / fp32_peak_tflops(mhz), 4),
            "direct_equiv_basis": "8 N_z flop per (particle, PA, component) over correlation + Gram kernel time, "
                                  "vs 74.45 TFLOP/s FP32: the direct method's flops, not executed by K1T",
            "achieved": None, "frac": None, "xu_frac": None, "traffic": None}
    rec = pipe_profile(args, cfg)
    # template instances are recorded with their full argument list (e.g. tay_gram_kernel<9, 1>: S, FAST path)
    match = [n for n in (rec or {}).get("kernels", {})
             if n == names[dom] or n.startswith(names[dom].rstrip(">") + ",") or n.startswith(names[dom] + "<")]
    if match:
        k = rec["kernels"][match[0]]
        roof["kernel"] = match[0]
        fma = k["fma_thread_inst_per_particle"] * P_local / launches_per_step
        xu = k["xu_thread_inst_per_particle"] * P_local / launches_per_step
        roof.update({"achieved": round(fma / t / 1e12, 3), "frac": round(fma / t / 1e12 / peak_fma, 4),
                     "xu_achieved": round(xu / t / 1e12, 3), "xu_frac": round(xu / t / 1e12 / peak_xu, 4),
                     "traffic": k.get("dram_bytes_per_particle", 0) * P_local / launches_per_step or None,
                     "traffic_basis": "dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full)",
                     "inst_source": rec["source"]})
    try:  # the pipe that actually limits the kernel (committed ncu --set full summary of this config)
        with open(os.path.join(ROOT, "profiles", "limiters.json")) as f:
            lim = json.load(f)
        k = lim.get(f"{args.config}_{args.wavefront}_{args.precision}", {}).get(roof["kernel"])
        if k:
            roof["limiter"] = {"pipe": k["pipe"], "pct_of_peak": k["pct_of_peak"], "fma_cycles_pct": k["fma_cycles_pct"],
                               "lsu_wavefronts_pct_of_peak": k["lsu_wavefronts_pct_of_peak"], "source": lim["source"]}
    except Exception:
        pass
    return roof


def kernel_names(args, cfg, P_local):
    """The likelihood stage's kernels as libcdms picks them (cdms.cpp engine selection, taylor.cu tay_lanes)."""
    if args.precision == "fp64" or os.environ.get("CDMS_TAYLOR", "1") == "0" and args.wavefront != "planar_nb":
        return {"corr": "corr_kernel", "gram": "(in corr_kernel)"}
    if args.wavefront == "planar_nb":
        return {"corr": "nb_corr_kernel", "gram": "nb_gram_kernel"}
    return {"corr": "tay_corr_lanes_kernel" if P_local * cfg.J < 250000 else "tay_corr_kernel",
            "gram": f"tay_gram_kernel<{cfg.S}>"}


def pipe_profile(args, cfg):
    """Per-particle pipe instruction counts of this config's kernels (tools/ncu_pipe.py from a committed capture)."""
    key = f"{args.config}_{args.wavefront}_{args.precision}"
    try:
        with open(os.path.join(ROOT, "profiles", "pipe_inst.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def fp32_weight_error(cdms, torch, dev):
    """Normalized weights of every c2 particle from the FP32 engine vs the oracle (identical inputs): max |dw|, max
    centred |dl| (dl minus its weighted mean), reading C-amb-18(ii)."""
    from oracle import oracle as O
    O.build()
    cfg = scenes.CONFIGS["c2"]
    sc = scenes.make_scene(cfg)
    o, y, eta, m, v, x = oracle_inputs(cfg, sc, O, cfg.P)
    t0 = time.perf_counter()
    st, lo = o.loglik(x, sc.sfv, y, m, v, eta)
    t_orc = time.perf_counter() - t0
    st, wo, lseo = O.normalize(lo)
    ctx = cdms.Context(int(dev.split(":")[1]))
    scene = cdms.Scene.from_synthetic(sc)
    l = cdms.loglik(ctx, scene, torch.as_tensor(x, device=dev).contiguous(),
                    torch.as_tensor(sc.sfv, device=dev).contiguous(),
                    torch.as_tensor(y.astype(np.complex64), device=dev).contiguous(), m, v, eta)
    w, lse = cdms.weights_normalize(ctx, l)
    ctx.sync()
    w = w.cpu().numpy()
    dl = l.cpu().numpy() - lo
    ctx.close()
    return {"config": "c2 (all 100000 particles)", "max_abs_dw": float(np.max(np.abs(w - wo))),
            "max_w": float(wo.max()), "max_centred_abs_dl": float(np.max(np.abs(dl - np.sum(wo * dl)))),
            "lse_gpu": float(lse.item()), "lse_oracle": float(lseo), "oracle_s": round(t_orc, 2)}


def fp64_mode_line(cdms, torch, dev, local, config="c2", steps=5):
    """Throughput of the FP64 engine (the mode whose weights meet 1e-5 end to end) on a BASELINE config."""
    cfg = scenes.CONFIGS[config]
    sc = scenes.make_scene(cfg)
    stream = torch.cuda.current_stream(local)
    ctx = cdms.Context(local, stream)
    scene = cdms.Scene.from_synthetic(sc, precision="fp64")
    y, eta = synth_measurement(cdms, ctx, scene, sc, torch, dev)
    m, v = scenes.priors(sc, "nzm")
    x = torch.as_tensor(scenes.make_particles(cfg), device=dev).contiguous()
    dsfv = torch.as_tensor(sc.sfv, device=dev).contiguous()
    for n in range(3):
        cdms.bp_step(ctx, scene, x, dsfv, y, m, v, eta, 0.1, 0.5, sc.philox_key, n)
    torch.cuda.synchronize(local)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for n in range(steps):
        cdms.bp_step(ctx, scene, x, dsfv, y, m, v, eta, 0.1, 0.5, sc.philox_key, 3 + n)
    b.record(stream)
    ctx.sync()
    ms = a.elapsed_time(b) / steps
    ctx.close()
    return {"config": f"{config}: J={cfg.J}, S={cfg.S}, {cfg.ny}x{cfg.nv}, nf={cfg.nf}, P={cfg.P}", "dtype": "f64",
            "ms_per_step": ms, "value": cfg.P * cfg.J * cfg.S / (ms / 1e3), "unit": UNIT, "steps": steps}


def oracle_inputs(cfg, sc, orc_mod, n_particles):
    o = orc_mod.Oracle.from_scene(sc)
    y, eta = orc_mod.measurement(o, sc, scenes.P_TRUE)
    y = y.astype(np.complex64).astype(np.complex128)
    m, v = scenes.priors(sc, "nzm")
    x = scenes.make_particles(cfg, 0, n_particles)
    return o, y, np.full(cfg.J, eta), m, v, x


def cpu_baseline(args, cfg, sc, budget_s: float = 15.0):
    """The oracle as it stands (fp64 C, OpenMP over particles) on this host's cores, on a bounded sample of
    the workload: time oracle BP steps on growing particle samples until ~budget_s of CPU work."""
    from oracle import oracle as O
    O.build()
    n = 64
    o, y, eta, m, v, x = oracle_inputs(cfg, sc, O, min(cfg.P, 64))
    spent, best = 0.0, None
    while True:
        xs = scenes.make_particles(cfg, 0, n)
        t0 = time.perf_counter()
        O.Oracle.bp_step(o, xs, sc.sfv, y, m, v, eta, 0.1, 0.5, sc.philox_key, 0)
        dt = time.perf_counter() - t0
        spent += dt
        best = (n, dt)
        if spent > budget_s or n >= cfg.P or dt > budget_s / 3:
            break
        n = min(cfg.P, n * 4)
    n, dt = best
    return {"value": n * cfg.J * cfg.S / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"oracle bp_step on {n} of {cfg.P} particles of {args.config} (fp64 C, OpenMP), {dt:.2f} s"}


def config_dict(args, cfg, P_total, world):
    """The workload both arms report (the reference arm times a bounded sample of it, stated in cpu_baseline)."""
    return {"workload": f"{args.config}: J={cfg.J} PAs, K={cfg.K} walls (S={cfg.S}), "
                        f"{cfg.ny}x{cfg.nv} URA, nf={cfg.nf}, P={P_total} total (strong scaling)",
            "config": args.config, "P_total": P_total, "P_per_gpu": P_total // world, "J": cfg.J,
            "K": cfg.K, "ny": cfg.ny, "nv": cfg.nv, "nf": cfg.nf, "Nz": cfg.Nz,
            "wavefront": args.wavefront, "precision": args.precision,
            "step": "predict+loglik+normalize+moments+resample+regularize",
            "l2": "flushed (256 MiB write) between timed steps; particles 48 B x P_total > L2",
            "parallelism": f"dp{world} (particles)"}


def run_reference(args):
    """--impl reference: the oracle as the reference arm, on this host's cores, bounded samples."""
    world, rank, local = dist_env()
    if rank != 0:
        return None
    from oracle import oracle as O
    O.build()
    cfg = scenes.CONFIGS[args.config]
    sc = scenes.make_scene(cfg)
    n = min(cfg.P, args.ref_particles)
    if n <= 0:  # auto: a per-step sample of ~ref_step_s of oracle work on this host (whole run within minutes)
        o, y, eta, m, v, x = oracle_inputs(cfg, sc, O, 16)
        t0 = time.perf_counter()
        O.Oracle.bp_step(o, x, sc.sfv, y, m, v, eta, 0.1, 0.5, sc.philox_key, 0)
        per = (time.perf_counter() - t0) / 16
        n = int(min(cfg.P, max(16, args.ref_step_s / max(per, 1e-9))))
    o, y, eta, m, v, x = oracle_inputs(cfg, sc, O, n)
    for w in range(args.warmup):
        O.Oracle.bp_step(o, x, sc.sfv, y, m, v, eta, 0.1, 0.5, sc.philox_key, w)
    times = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        O.Oracle.bp_step(o, x, sc.sfv, y, m, v, eta, 0.1, 0.5, sc.philox_key, args.warmup + k)
        times.append(time.perf_counter() - t0)
    dt = sum(times) / len(times)
    value = n * cfg.J * cfg.S / dt
    sample = f"oracle bp_step on {n} of {cfg.P} particles of {args.config} per step (fp64 C, OpenMP)"
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(args, cfg, p_total_of(args, cfg), world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


PF_METRIC = "PF particle x PA kappa~ update evals/s (F1)"
PF_UNIT = "PF particle-PA evals/s"


def pf_inputs(cfg, sc, P, rank=0):
    """One legacy PF (wall 1) of the synthetic scene: PF particles around its true SFV (+-5 cm) paired with MT particles
    of the config's mixture; the other K - 1 walls as the columns of M and the summed mean (scaled by sqrt(0.05) and
    0.9 rho_s: tests/test_pf_gpu.py's recipe).  Returns host arrays."""
    rng = np.random.default_rng(cfg.seed + 7 + rank)
    x = scenes.make_particles(cfg, rank * P, P)
    phi = sc.sfv[0][None, :] + 0.05 * rng.standard_normal((P, 3))
    walpha = np.full(P, 0.9 / P)
    mu = sc.rho[1] * (1 + 0.1 * (rng.standard_normal(P) + 1j * rng.standard_normal(P)))
    gamma = np.full(P, 0.02)
    return x, phi, walpha, mu, gamma, np.full(cfg.J, 0.9)


def run_pf(args):
    """F1: time cdms_pf_update for one PF with P PF particles (device-resident inputs), L = K - 1 other features."""
    import torch
    world, rank, local = dist_env()
    from paper_2604_19723_b200 import cdms
    dev = f"cuda:{local}"
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream(local)
    cfg = scenes.CONFIGS[args.config]
    P = p_total_of(args, cfg) // world
    sc = scenes.make_scene(cfg)
    scene = cdms.Scene.from_synthetic(sc, wavefront=args.wavefront, precision=args.precision)
    ctx = cdms.Context(local, stream)
    y, eta = synth_measurement(cdms, ctx, scene, sc, torch, dev)
    L = cfg.K - 1
    J = cfg.J
    pos = np.repeat(scenes.P_TRUE[None], J * L, axis=0)
    js = np.array([(j, 2 + l) for j in range(J) for l in range(L)], dtype=np.int32)
    psi = cdms.response(ctx, scene, pos, js, sc.sfv).reshape(J, L, -1)
    mcols = (math.sqrt(0.05) * psi).to(torch.complex64).reshape(J, L, cfg.nf, cfg.Na).contiguous()
    rho = torch.as_tensor(sc.rho[2:2 + L], device=dev)
    mu3 = (0.9 * torch.einsum("jln,l->jn", psi, rho)).to(torch.complex64).reshape(J, cfg.nf, cfg.Na).contiguous()
    x, phi, wa, mu, gamma, zeta = pf_inputs(cfg, sc, P, rank)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
    dx, dphi, dwa, dmu, dg = t(x), t(phi), t(wa), t(mu.astype(np.complex128)), t(gamma)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        return cdms.pf_update(ctx, scene, dx, dphi, dwa, dmu, dg, zeta, eta, y, mu3, mcols)

    for _ in range(args.warmup):
        step()
    ctx.sync()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(local)
        for n in range(args.steps):
            flush.zero_()
            ev[n][0].record(stream)
            step()
            ev[n][1].record(stream)
        clk.mark()
        torch.cuda.synchronize(local)
    st = ctx.sync(raise_on_error=False)
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    evals = P * J * world
    res = {"metric": PF_METRIC, "value": evals / (ms / 1e3), "unit": PF_UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f32", "data": "synthetic",
           "config": {"workload": f"{args.config} scene (J={J}, {cfg.ny}x{cfg.nv}, nf={cfg.nf}), one PF with {P} "
                                  f"particles/GPU, L={L} other features", "config": args.config, "mode": "pf",
                      "P_per_gpu": P, "L": L, "Nz": cfg.Nz, "wavefront": args.wavefront,
                      "step": "snapshots + fp64 factor of A + K1T tables of L+1 snapshots + per-particle "
                              "correlations + rank-1 lemma + M_y normalization"},
           "clocks": clk.summary(), "gpu_launches": ctx.launch_count() - launches0, "sync_status": st}
    ctx.close()
    if not args.no_cpu_baseline and rank == 0:
        from oracle import oracle as O
        O.build()
        o = O.Oracle.from_scene(sc, wavefront=args.wavefront)
        n = 8
        while True:
            t0 = time.perf_counter()
            o.pf_update(x[:n], phi[:n], wa[:n], mu[:n], gamma[:n], zeta, eta, y.cpu().numpy().astype(np.complex128),
                        mu3.cpu().numpy().astype(np.complex128), mcols.cpu().numpy().astype(np.complex128))
            dt = time.perf_counter() - t0
            if dt > args.cpu_seconds / 3 or n >= P:
                break
            n = min(P, n * 4)
        res["cpu_baseline"] = {"value": n * J / dt, "unit": PF_UNIT, "cores": 1, "kind": "oracle",
                               "sample": f"orc_pf_update on {n} of {P} PF particles ({args.config}), {dt:.2f} s"}
    return res if rank == 0 else None


SLAM_METRIC = "SLAM time steps x paired particles/s (F4)"
SLAM_UNIT = "particle-steps/s"


def run_slam(args):
    """F4: time cdms_slam_step on an Experiment-1-shaped track (tools/slam_run.py's scene and start, a rough prior map:
    the LOS and every wall as PFs, so every step runs all S slots' messages plus one birth).  The snapshots of the
    W + K steps are synthesized before the timed region (device-resident); the state (P paired particles, > L2) is
    the library's."""
    import torch
    world, rank, local = dist_env()
    if world > 1:
        raise SystemExit("--mode slam: the F4 driver is single-rank (DESIGN.md section 8e)")
    from paper_2604_19723_b200 import cdms
    dev = f"cuda:{local}"
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream(local)
    cfg = scenes.CONFIGS[args.config]
    P = args.particles if args.particles is not None else 1_000_000
    sc = scenes.make_scene(cfg)
    scene = cdms.Scene.from_synthetic(sc, wavefront=args.wavefront, precision=args.precision)
    ctx = cdms.Context(local, stream)
    J, S = cfg.J, cfg.S
    T = 0.1
    n_all = args.warmup + args.steps
    js = np.array([(j, s) for j in range(J) for s in range(S)], dtype=np.int32)
    rho = torch.as_tensor(sc.rho, device=dev)
    gen = torch.Generator(device=dev).manual_seed(cfg.seed)
    ys, eta = [], None
    for n in range(1, n_all + 1):
        p = scenes.P_TRUE + scenes.V_TRUE * T * n
        psi = cdms.response(ctx, scene, np.repeat(p[None], J * S, axis=0), js, sc.sfv).reshape(J, S, -1)
        clean = torch.einsum("jsn,s->jn", psi, rho)
        if eta is None:
            eta = float((clean.abs() ** 2).sum().item()) / (scene.Nz * J) / 100.0
        w = torch.complex(torch.randn(clean.shape, generator=gen, device=dev, dtype=torch.float64),
                          torch.randn(clean.shape, generator=gen, device=dev, dtype=torch.float64)) / math.sqrt(2.0)
        ys.append((clean + math.sqrt(eta) * w).to(torch.complex64).reshape(J, cfg.nf, cfg.Na).contiguous())
    slam = cdms.Slam(ctx, scene, P, T=T, box=(-10.0, -5.0, -4.0, 12.0, 12.0, 6.0))
    rng = np.random.default_rng(cfg.seed)
    x0 = np.zeros((P, 6))
    x0[:, :3] = scenes.P_TRUE + 0.1 * rng.standard_normal((P, 3))
    x0[:, 3:] = scenes.V_TRUE + 0.1 * rng.standard_normal((P, 3))
    slam.init(torch.as_tensor(x0, device=dev), torch.full((J, P), eta, dtype=torch.float64, device=dev))
    v = slam.view()
    for s_ in range(1, S):
        v["phi"][s_].copy_(torch.as_tensor(sc.sfv[s_ - 1][None, :] + 0.05 * rng.standard_normal((P, 3))))
    for s_ in range(S):
        v["mu"][s_].fill_(complex(sc.rho[s_]))
        v["gamma"][s_].fill_(0.01)
        v["w"][s_].fill_(0.9 / P)
    slam.set_slots(list(range(S)), np.full((S, J), 0.9), np.vstack([np.zeros(3), sc.sfv]), n=1, next_id=S)
    for n in range(args.warmup):
        slam.step(ys[n])
    ctx.sync()
    launches0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    feats = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(local)
        ev0.record(stream)
        for n in range(args.warmup, n_all):
            r = slam.step(ys[n])
            feats.append(r["n_feat"])
        ev1.record(stream)
        clk.mark()
        torch.cuda.synchronize(local)
    st = ctx.sync(raise_on_error=False)
    ms = ev0.elapsed_time(ev1) / args.steps
    last = r
    err = float(np.linalg.norm(last["est"][1:4] - (scenes.P_TRUE + scenes.V_TRUE * T * n_all)))
    # e2e: the same steps with each snapshot copied from pinned host memory inside the timed region
    yh = [y.cpu().pin_memory() for y in ys[args.warmup:]]
    yd = torch.empty_like(ys[0])
    t0 = time.perf_counter()
    for n in range(args.steps):
        yd.copy_(yh[n], non_blocking=True)
        slam.step(yd)
    torch.cuda.synchronize(local)
    ms_e2e = (time.perf_counter() - t0) * 1e3 / args.steps
    # the paper's full SLAM step of Experiment 1 (this scene shape, P = 30 000) took 400 ms on an RTX PRO
    # 4000 Blackwell -- another machine's number, context only; quoted only for exactly that workload
    vs = (P / (ms / 1e3)) / (30000 / 0.400) if (args.config == "exp1" and P == 30000) else None
    res = {"metric": SLAM_METRIC, "value": P / (ms / 1e3), "unit": SLAM_UNIT, "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": vs,
           "dtype": "f32" if args.precision == "fp32" else "f64", "data": "synthetic",
           "config": {"workload": f"{args.config} scene (J={J}, {cfg.ny}x{cfg.nv}, nf={cfg.nf}, K={cfg.K}), F4 step "
                                  f"with {P} paired particles, LOS + {cfg.K} PF slots + one birth per step",
                      "config": args.config, "mode": "slam", "P": P, "slots_per_step": sorted(set(feats)),
                      "l2": "state > L2 (P paired particles over all slots)",
                      "step": "transitions + birth (F3) + belief columns + iota~ + nu~ + kappa~/omega~ per slot + "
                              "resampling + SFV regularization + estimates / pruning (4 host syncs)"},
           "final_position_error_m": err,
           "e2e": {"value": P / (ms_e2e / 1e3), "unit": SLAM_UNIT, "ms_per_step": ms_e2e,
                   "h2d_bytes_per_step": int(ys[0].numel() * 8), "d2h_bytes_per_step": 0},
           "clocks": clk.summary(), "gpu_launches": ctx.launch_count() - launches0, "sync_status": st}
    slam.close()
    ctx.close()
    if not args.no_cpu_baseline:
        from oracle import oracle as O
        from oracle import slam as OS
        O.build()
        base = O.Oracle.from_scene(sc, wavefront=args.wavefront)
        prm = OS.Params(T=T, box=(-10.0, -5.0, -4.0, 12.0, 12.0, 6.0))
        n = 64
        while True:
            xs = x0[:n].copy()
            st0 = OS.State(xs, np.full((J, n), eta), [OS.init_los(n, J, prm)])
            t0 = time.perf_counter()
            OS.step(base, st0, ys[0].cpu().numpy().astype(np.complex128), prm)
            dt = time.perf_counter() - t0
            if dt > args.cpu_seconds / 3 or n >= 4096:
                break
            n *= 4
        res["cpu_baseline"] = {"value": n / dt, "unit": SLAM_UNIT, "cores": 1, "kind": "oracle",
                               "sample": f"oracle/slam.py step from the LOS alone with {n} paired particles "
                                         f"({args.config}), {dt:.2f} s"}
    return res


BIRTH_METRIC = "Bartlett birth-proposal candidate x PA correlations/s (F3)"
BIRTH_UNIT = "candidate-PA evals/s"


def birth_inputs(cfg, sc, L):
    """x_hat near the truth, the first L walls as legacy PFs, the partition box around the next wall (+-0.4 m)."""
    x_hat = scenes.P_TRUE + np.array([0.01, -0.02, 0.005])
    target = sc.sfv[min(L, cfg.K - 1)]
    return x_hat, sc.sfv[:L], np.concatenate([target - 0.4, target + 0.4])


def birth_config(args, cfg, world):
    return {"workload": f"{args.config} scene (J={cfg.J}, {cfg.ny}x{cfg.nv} URA, nf={cfg.nf}), birth proposal with "
                        f"L={args.legacy} legacy PFs, N_g={args.candidates} candidates/GPU",
            "config": args.config, "mode": "birth", "N_g_per_gpu": args.candidates, "L": args.legacy, "J": cfg.J,
            "Nz": cfg.Nz, "wavefront": args.wavefront, "precision": args.precision,
            "step": "residual projector + candidates + coherent Bartlett correlations + mode/moment matching",
            "l2": "flushed (256 MiB write) between timed steps", "parallelism": f"replicas x{world} (independent draws)"}


def run_birth(args):
    """F3: time cdms_birth_proposal (device-resident snapshot) and its end-to-end variant (pinned host snapshot
    uploaded and the 13-double result read back every step)."""
    import torch
    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_2604_19723_b200 import build as B
    if rank == 0 and not os.path.exists(os.path.join(ROOT, "paper_2604_19723_b200", "libcdms.so")):
        B.build()
    if world > 1:
        torch.distributed.barrier()
    from paper_2604_19723_b200 import cdms
    dev = f"cuda:{local}"
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream(local)
    cfg = scenes.CONFIGS[args.config]
    sc = scenes.make_scene(cfg)
    scene = cdms.Scene.from_synthetic(sc, wavefront=args.wavefront, precision=args.precision)
    ctx = cdms.Context(local, stream)
    y, _ = synth_measurement(cdms, ctx, scene, sc, torch, dev)
    x_hat, sl, box = birth_inputs(cfg, sc, args.legacy)
    N_g = args.candidates
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    out = torch.empty(13, dtype=torch.float64, device=dev)
    key = sc.philox_key

    def step(n):
        return cdms.birth_proposal(ctx, scene, x_hat, sl, y, box, N_g, key, 1000 * rank + n, want_pb=False,
                                   want_cand=False)

    def barrier():
        torch.cuda.synchronize(local)
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize(local)

    for n in range(args.warmup):
        step(n)
    ctx.sync()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    ctx.timing_enable(True)
    with ClockSampler(local) as clk:
        barrier()
        for n in range(args.steps):
            flush.zero_()
            ev[n][0].record(stream)
            step(args.warmup + n)
            ev[n][1].record(stream)
            if n == args.steps // 2:
                clk.mark()
        clk.mark()
        barrier()
    st = ctx.sync(raise_on_error=False)
    gpu_launches = ctx.launch_count() - launches0
    k_ms, k_n = ctx.timing_read()
    ctx.timing_enable(False)
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_per_step = t.item() / args.steps
    kernel_ms = k_ms / max(k_n, 1)
    launches_per_step = k_n / args.steps
    # end to end: pinned host snapshot -> device, proposal, result -> pinned host
    y_host = y.cpu().pin_memory()
    out_host = torch.empty(13, dtype=torch.float64).pin_memory()
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    for n in range(args.steps):
        flush.zero_()
        e2e_ev[n][0].record(stream)
        y.copy_(y_host, non_blocking=True)
        o, _, _ = step(10_000 + n)
        out_host.copy_(o, non_blocking=True)
        e2e_ev[n][1].record(stream)
    barrier()
    te = torch.tensor([sum(a.elapsed_time(b) for a, b in e2e_ev)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_ms = te.item() / args.steps
    ctx.sync(raise_on_error=False)
    evals = N_g * cfg.J * world
    result = None
    if rank == 0:
        clocks = clk.summary()
        flop_launch = 8.0 * cfg.Nz * N_g * cfg.J / launches_per_step
        if nb_tensor_path(args):
            t_peak, t_basis = measured_tensor_peak()
            ach = 4.0 * flop_launch / (kernel_ms / 1e3) / 1e12
            roof = {"bound": "tensor", "pipe": "tcgen05.mma kind::f16", "achieved": round(ach, 2),
                    "peak": round(t_peak, 1), "unit": "TFLOP/s", "frac": round(ach / t_peak, 4), "peak_basis": t_basis,
                    "kernel": "cdms::nb_corr_kernel (F3 correlations)"}
        else:
            ach = flop_launch / (kernel_ms / 1e3) / 1e12
            peak = fp32_peak_tflops(1965.0)
            roof = {"bound": "alu", "pipe": "fp32 (direct-correlation flop equivalent)" if taylor_path(args)
                    else "fp32 fma", "achieved": round(ach, 3), "peak": round(peak, 2),
                    "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                    "peak_basis": "128 FFMA/SM/clk x 148 SM x 2 FLOP x 1965 MHz (sm_max); DESIGN.md 'Roofline'",
                    "kernel": (("cdms::tay_corr_lanes_kernel" if (N_g // 8) * cfg.J < 250000
                                else "cdms::tay_corr_kernel") + " (K1T, F3 correlations of the candidate walls, 8 "
                               "candidates per pseudo-particle)" if taylor_path(args)
                               else "cdms::corr_kernel (F3 correlations of the candidate walls)")}
            if taylor_path(args):
                roof["note"] = ("frac > 1: K1T evaluates the correlations from spectral Taylor tables; the flop count "
                                "is the direct correlation's 8 N_z per (candidate, PA)")
        roof.update({"kernel_ms": round(kernel_ms, 4), "kernel_share_of_step": round(kernel_ms * launches_per_step /
                                                                                    ms_per_step, 4),
                     "launches_per_step": launches_per_step,
                     "flop_basis": "8 N_z flop per (candidate, PA): one complex MAC per response element",
                     "traffic": None})
        result = {"metric": BIRTH_METRIC, "value": evals / (ms_per_step / 1e3), "unit": BIRTH_UNIT, "n_gpus": world,
                  "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                  "scaling": "weak", "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
                  "data": "synthetic", "config": birth_config(args, cfg, world), "roofline": roof,
                  "e2e": {"value": evals / (e2e_ms / 1e3), "unit": BIRTH_UNIT, "ms_per_step": e2e_ms,
                          "h2d_bytes_per_step": int(y.numel() * 8), "d2h_bytes_per_step": 13 * 8},
                  "clocks": clocks, "gpu_launches": int(gpu_launches), "sync_status": st}
        if not args.no_cpu_baseline:
            result["cpu_baseline"] = birth_cpu_baseline(args, cfg, sc, args.cpu_seconds)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return result


def birth_cpu_baseline(args, cfg, sc, budget_s):
    """The oracle's orc_birth_proposal on growing candidate samples until ~budget_s of CPU work (single thread:
    the oracle's candidate loop is serial)."""
    from oracle import oracle as O
    O.build()
    o = O.Oracle.from_scene(sc, wavefront=args.wavefront)
    y, _ = O.measurement(o, sc, scenes.P_TRUE)
    y = y.astype(np.complex64).astype(np.complex128).reshape(cfg.J, -1)
    x_hat, sl, box = birth_inputs(cfg, sc, args.legacy)
    n, spent, best = 16, 0.0, None
    while True:
        t0 = time.perf_counter()
        o.birth_proposal(x_hat, sl, y, box, n, sc.philox_key, 0)
        dt = time.perf_counter() - t0
        spent += dt
        best = (n, dt)
        if spent > budget_s or dt > budget_s / 3 or n >= args.candidates:
            break
        n = min(args.candidates, n * 4)
    n, dt = best
    return {"value": n * cfg.J / dt, "unit": BIRTH_UNIT, "cores": 1, "kind": "oracle",
            "sample": f"orc_birth_proposal with {n} of {args.candidates} candidates ({args.config}), {dt:.2f} s"}


def run_birth_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return None
    from oracle import oracle as O
    O.build()
    cfg = scenes.CONFIGS[args.config]
    sc = scenes.make_scene(cfg)
    o = O.Oracle.from_scene(sc, wavefront=args.wavefront)
    y, _ = O.measurement(o, sc, scenes.P_TRUE)
    y = y.astype(np.complex64).astype(np.complex128).reshape(cfg.J, -1)
    x_hat, sl, box = birth_inputs(cfg, sc, args.legacy)
    n = min(args.candidates, args.ref_particles)
    for w in range(args.warmup):
        o.birth_proposal(x_hat, sl, y, box, n, sc.philox_key, w)
    times = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        o.birth_proposal(x_hat, sl, y, box, n, sc.philox_key, args.warmup + k)
        times.append(time.perf_counter() - t0)
    dt = sum(times) / len(times)
    value = n * cfg.J / dt
    return {"metric": BIRTH_METRIC, "value": value, "unit": BIRTH_UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": birth_config(args, cfg, world),
            "cpu_baseline": {"value": value, "unit": BIRTH_UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"orc_birth_proposal with {n} of {args.candidates} candidates per step"},
            "e2e": {"value": value, "unit": BIRTH_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(scenes.CONFIGS))
    ap.add_argument("--particles", type=int, default=None,
                    help="P_total over all GPUs, strong scaling (default: the config's P; c5: 16M)")
    ap.add_argument("--wavefront", default="spherical", choices=["spherical", "planar_wb", "planar_nb"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--impl", default="cdms", choices=["cdms", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the FP32-weights-vs-oracle and FP64-mode fields")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-particles", type=int, default=0,
                    help="--impl reference: particles per oracle step (0: sized to ~--ref-step-s seconds per step)")
    ap.add_argument("--ref-step-s", type=float, default=2.0)
    ap.add_argument("--mode", default="step", choices=["step", "birth", "pf", "slam"],
                    help="step: the BP step (headline); birth: the F3 birth proposal; pf: F1; slam: the F4 step")
    ap.add_argument("--candidates", type=int, default=1 << 20, help="birth mode: candidates N_g per GPU")
    ap.add_argument("--legacy", type=int, default=2, help="birth mode: legacy PFs L")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "cdms" else args.warmup
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.mode == "birth":
        res = run_birth_reference(args) if args.impl == "reference" else run_birth(args)
    elif args.mode == "pf":
        res = None if args.impl == "reference" else run_pf(args)
    elif args.mode == "slam":
        res = None if args.impl == "reference" else run_slam(args)
    else:
        res = run_reference(args) if args.impl == "reference" else run_cdms(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
