"""GPU parity: libcdms (CUDA, through the C ABI) against the fp64 oracle on identical seeded inputs.

Tolerances (north_star; readings C-amb-11/18 in DESIGN.md):
  * response phase |arg(psi_gpu conj psi_orc)| <= 1e-4 rad per element (FP32), 1e-9 (FP64);
  * rel-l = |l_gpu - l_orc| / max(|l_orc|, J Nz) <= 1e-4 (FP32), 1e-10 (FP64);
  * normalized weights within 1e-5 (given identical l, and end to end in FP64 mode);
  * resampled ancestors bit-exact given identical (w, u_bits).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2604_19723_b200 import scenes
from tests.gpu_common import Case, record, rel_err
from tests.helpers import small_cfg, wrap


@pytest.fixture(scope="module")
def cd():
    from paper_2604_19723_b200 import build as B
    B.build()
    from paper_2604_19723_b200 import cdms
    return cdms


@pytest.fixture(scope="module")
def ctx(cd):
    c = cd.Context(0)
    yield c
    c.close()


# FP64 bound: the fp64 evaluation itself is conditioned by
# kappa(K) * u * (||e||^2/eta) / (J Nz) ~ (1 + v Nz/eta) * 1.1e-16 * SNR ~ 1e-9 at the configs' scale,
# on the oracle side as well; 1e-8 leaves a margin above that floor.
TOL_L = {"fp32": 1e-4, "fp64": 1e-8}
TOL_PH = {"fp32": 1e-4, "fp64": 1e-9}


# ---------------------------------------------------------------------------- A1 layout
def test_layout_parity(cd, ctx, orc):
    sc = scenes.make_scene(scenes.CONFIGS["c5"])
    o = orc.Oracle.from_scene(sc)
    scene = cd.Scene.from_synthetic(sc)
    lay, va, H = cd.layout(ctx, scene, sc.sfv)
    ctx.sync()
    st, lay_o, va_o, H_o = o.layout(sc.sfv)
    assert np.allclose(lay.cpu().numpy(), lay_o, atol=1e-12, rtol=0)
    assert np.allclose(va.cpu().numpy(), va_o, atol=1e-12, rtol=0)
    assert np.allclose(H.cpu().numpy(), H_o, atol=1e-14, rtol=0)


# ---------------------------------------------------------------------------- A2 responses
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("wf", ["spherical", "planar_wb", "planar_nb"])
@pytest.mark.parametrize("shape", [(4, 4, 16, 2), (8, 8, 1024, 8), (16, 16, 256, 4), (3, 5, 100, 3)])
def test_response_phase_parity(cd, ctx, orc, precision, wf, shape):
    ny, nv, nf, K = shape
    cfg = small_cfg(J=2, K=K, ny=ny, nv=nv, nf=nf)
    sc = scenes.make_scene(cfg)
    o = orc.Oracle.from_scene(sc, wavefront=wf)
    scene = cd.Scene.from_synthetic(sc, wavefront=wf, precision=precision)
    rng = np.random.default_rng(11)
    pos, js = [], []
    for t in range(6):
        p = scenes.ROI_LO + (scenes.ROI_HI - scenes.ROI_LO) * rng.uniform(size=3)
        for j in range(2):
            for s in range(K + 1):
                pos.append(p)
                js.append((j, s))
    psi = cd.response(ctx, scene, np.array(pos), np.array(js), sc.sfv)
    ctx.sync()
    psi = psi.cpu().numpy()
    worst_ph, worst_mag = 0.0, 0.0
    for i, (p, (j, s)) in enumerate(zip(pos, js)):
        st, ref = o.response(p, j, s, sc.sfv)
        assert st == 0
        worst_ph = max(worst_ph, np.max(np.abs(np.angle(psi[i] * np.conj(ref)))))
        worst_mag = max(worst_mag, np.max(np.abs(np.abs(psi[i]) - 1.0)))
    record("phase_rad", worst_ph, TOL_PH[precision], precision=precision, wavefront=wf, shape=list(shape))
    record("magnitude", worst_mag, TOL_PH[precision], precision=precision, wavefront=wf, shape=list(shape))
    assert worst_ph <= TOL_PH[precision], worst_ph
    assert worst_mag <= TOL_PH[precision], worst_mag


# ---------------------------------------------------------------------------- A3-A5 log-likelihood
def check_loglik(case, ctx, precision, idx=None, amp=False):
    l = case.gpu_loglik(ctx, want_amp=amp)
    if amp:
        l, a = l
    ctx.sync()
    l = l.cpu().numpy()
    if idx is None:
        idx = np.arange(case.x.shape[0])
    res = case.oracle_loglik(idx, want_amp=amp)
    lo = res[1]
    assert res[0] == 0
    e = rel_err(l[idx], lo, case.cfg.J, case.cfg.Nz)
    record("rel_l", e.max(), TOL_L[precision], precision=precision, config=case.cfg.name, n=int(len(idx)))
    assert np.all(np.isfinite(l[idx]))
    assert e.max() <= TOL_L[precision], (e.max(), int(np.argmax(e)))
    if amp:
        ga = a.cpu().numpy()[idx]
        scale = np.abs(res[2]).max()
        assert np.max(np.abs(ga - res[2])) <= (1e-3 if precision == "fp32" else 1e-9) * scale
    return l, e


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("wf", ["spherical", "planar_wb", "planar_nb"])
def test_loglik_c1_all_particles(cd, ctx, orc, precision, wf):
    case = Case(orc, scenes.CONFIGS["c1"], wavefront=wf, precision=precision)
    check_loglik(case, ctx, precision, amp=True)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("shape", [
    dict(J=2, K=3, ny=3, nv=5, nf=100, P=77),        # ragged antennas (15), ragged segment, ragged tile
    dict(J=3, K=0, ny=2, nv=2, nf=300, P=65),        # S = 1, two chunks, ragged chunk
    dict(J=1, K=8, ny=8, nv=8, nf=520, P=40),        # S = 9, 3 chunks, ragged segment
    dict(J=8, K=1, ny=1, nv=1, nf=1, P=33),          # single element, single subcarrier, J = 8 (the ABI maximum)
    dict(J=1, K=5, ny=16, nv=16, nf=64, P=31),       # 32 antenna blocks
])
def test_loglik_ragged_shapes(cd, ctx, orc, precision, shape):
    cfg = small_cfg(**shape, index=97)
    case = Case(orc, cfg, precision=precision)
    check_loglik(case, ctx, precision, amp=True)


def test_loglik_zm_and_pathloss(cd, ctx, orc):
    cfg = small_cfg(J=2, K=2, nf=64)
    check_loglik(Case(orc, cfg, mode="zm"), ctx, "fp32")
    check_loglik(Case(orc, cfg, pathloss=True), ctx, "fp32")
    check_loglik(Case(orc, cfg, pathloss=True, wavefront="planar_nb", precision="fp64"), ctx, "fp64")


def test_loglik_sfv_per_particle_and_prior(cd, ctx, orc):
    import torch
    cfg = small_cfg(J=2, K=3, nf=32, P=70)
    case = Case(orc, cfg)
    rng = np.random.default_rng(3)
    sfv_pp = case.sc.sfv[None] * (1.0 + 0.05 * rng.standard_normal((cfg.P, cfg.K, 3)))
    lw = rng.normal(size=cfg.P)
    d_sfv = torch.as_tensor(sfv_pp, device="cuda:0").contiguous()
    d_lw = torch.as_tensor(lw, device="cuda:0").contiguous()
    l = cd.loglik(ctx, case.scene, case.dx, d_sfv, case.dy, case.m, case.v, case.eta, logw_prior=d_lw,
                  sfv_per_particle=True)
    ctx.sync()
    st, lo = case.o.loglik(case.x, sfv_pp, case.y, case.m, case.v, case.eta, logw_prior=lw, sfv_per_particle=True)
    assert rel_err(l.cpu().numpy(), lo, cfg.J, cfg.Nz).max() <= 1e-4


def test_loglik_degenerate_and_invalid(cd, ctx, orc):
    import torch
    cfg = small_cfg(J=1, K=1, nf=16, P=40)
    case = Case(orc, cfg)
    x = case.x.copy()
    x[7, :3] = case.sc.pa_pos[0]      # MT on the PA phase centre
    case.dx = torch.as_tensor(x, device="cuda:0").contiguous()
    l = case.gpu_loglik(ctx)
    with pytest.raises(cd.CdmsError) as ei:
        ctx.sync()
    assert ei.value.status == cd.EDEGENERATE
    l = l.cpu().numpy()
    assert l[7] == -np.inf and np.all(np.isfinite(np.delete(l, 7)))
    # host-checkable problems -> EINVAL before any launch
    bad = cd.Scene(case.sc.pa_pos, case.sc.pa_rot * 1.01, cfg.ny, cfg.nv, case.sc.dy, case.sc.dv, cfg.nf,
                   cfg.fc, cfg.df, cfg.K)
    with pytest.raises(cd.CdmsError) as ei:
        cd.loglik(ctx, bad, case.dx, case.dsfv, case.dy, case.m, case.v, case.eta)
    assert ei.value.status == cd.EINVAL
    with pytest.raises(cd.CdmsError):
        cd.loglik(ctx, case.scene, case.dx, case.dsfv, case.dy, case.m, -case.v, case.eta)
    with pytest.raises(cd.CdmsError):
        cd.loglik(ctx, case.scene, case.dx, case.dsfv, case.dy, case.m, case.v, 0 * case.eta)
    # ||sfv|| = 0 is detected on the device -> EINVAL at sync
    zero = torch.zeros_like(case.dsfv)
    cd.loglik(ctx, case.scene, case.dx, zero, case.dy, case.m, case.v, case.eta)
    with pytest.raises(cd.CdmsError) as ei:
        ctx.sync()
    assert ei.value.status == cd.EINVAL


def test_loglik_placement_independent(cd, ctx, orc):
    """Per-particle results are bitwise independent of batch position and batch size."""
    import torch
    cfg = small_cfg(J=2, K=4, ny=8, nv=8, nf=128, P=300)
    case = Case(orc, cfg)
    l_full = case.gpu_loglik(ctx).cpu().numpy()
    perm = np.random.default_rng(0).permutation(cfg.P)[:123]
    sub = torch.as_tensor(case.x[perm], device="cuda:0").contiguous()
    l_sub = cd.loglik(ctx, case.scene, sub, case.dsfv, case.dy, case.m, case.v, case.eta).cpu().numpy()
    ctx.sync()
    assert np.array_equal(l_sub, l_full[perm])


@pytest.mark.parametrize("name,wf,nsample", [
    ("c2", "spherical", 1024),
    ("c3", "spherical", 256),
    ("c4", "spherical", 128),
    ("c4", "planar_wb", 128),
    ("c4", "planar_nb", 128),
    ("c2", "planar_nb", 512),    # F2 tensor-core path at the bench configurations
    ("c3", "planar_nb", 128),
])
def test_loglik_full_size_sampled(cd, ctx, orc, name, wf, nsample):
    """Full BASELINE sizes in the bench launch configuration; oracle on a stratified sample."""
    cfg = scenes.CONFIGS[name]
    case = Case(orc, cfg, wavefront=wf)
    idx = scenes.stratified_sample(cfg.P, nsample)
    l, e = check_loglik(case, ctx, "fp32", idx=idx)
    assert np.all(np.isfinite(l))


@pytest.mark.parametrize("name,wf", [("c2", "spherical"), ("c3", "spherical"), ("c4", "planar_nb"),
                                     ("c2", "planar_nb"), ("c3", "planar_nb"),
                                     ("c4", "spherical"), ("c5", "spherical")])
def test_loglik_near_truth_worst_case(cd, ctx, orc, name, wf):
    """Particles within 1 mm of the true position: ||e||^2 = ||z||^2 - 2 Re(m^H c) + m^H G m cancels by
    ~SNR there, the most demanding case for the fp32 correlation."""
    cfg = scenes.CONFIGS[name]
    rng = np.random.default_rng(17)
    x = np.zeros((32, 6))
    x[:, :3] = scenes.P_TRUE[None] + rng.uniform(-1e-3, 1e-3, size=(32, 3))
    x[0, :3] = scenes.P_TRUE
    case = Case(orc, cfg, wavefront=wf, particles=x)
    check_loglik(case, ctx, "fp32", idx=np.arange(8))


@pytest.mark.parametrize("P", [4096, 300_000])
def test_taylor_layouts_near_truth(cd, ctx, orc, P):
    """K1T picks its table layout and correlation kernel from P J (taylor.cu tay_lanes: lane groups with the
    [g][h][m] table below 250k, one thread per particle with the [m][g][l] table above); both at the near-truth
    worst case, plus a stratified sample."""
    import dataclasses
    cfg = dataclasses.replace(scenes.CONFIGS["c2"], P=P)  # c2's scene, P particles
    rng = np.random.default_rng(23)
    x = scenes.make_particles(cfg)
    x[:32, :3] = scenes.P_TRUE[None] + rng.uniform(-1e-3, 1e-3, size=(32, 3))
    case = Case(orc, cfg, wavefront="spherical", particles=x)
    idx = np.unique(np.concatenate([np.arange(8), scenes.stratified_sample(P, 64)]))
    check_loglik(case, ctx, "fp32", idx=idx)


def test_loglik_c5_shard_sampled(cd, ctx, orc):
    """c5 (J=4, S=9, Nz=65536) on one rank's 8-GPU shard (2M particles), oracle on 96 particles."""
    cfg = scenes.CONFIGS["c5"]
    P = cfg.P // 8
    case = Case(orc, cfg, P=P)
    idx = scenes.stratified_sample(P, 96)
    check_loglik(case, ctx, "fp32", idx=idx)


# ---------------------------------------------------------------------------- A6-A8
def test_normalize_moments_parity(cd, ctx, orc):
    import torch
    rng = np.random.default_rng(4)
    for P in [1, 31, 2049, 100_000]:
        l = rng.normal(-1e5, 30.0, P)
        l[rng.uniform(size=P) < 0.05] = -np.inf
        if P == 1:
            l[0] = -3.0
        dl = torch.as_tensor(l, device="cuda:0")
        w, lse = cd.weights_normalize(ctx, dl)
        x = rng.normal(size=(P, 6))
        est = cd.moments(ctx, torch.as_tensor(x, device="cuda:0"), w)
        ctx.sync()
        st, wo, lseo = orc.normalize(l)
        w = w.cpu().numpy()
        record("normalize_weights_abs", np.max(np.abs(w - wo)), 1e-12 * max(1.0, wo.max()), P=P)
        assert abs(lse.item() - lseo) <= 1e-12 * abs(lseo)
        assert np.max(np.abs(w - wo)) <= 1e-12 * max(1.0, wo.max())
        assert abs(w.sum() - 1.0) <= 1e-12
        st, esto = orc.moments(x, wo)
        assert np.allclose(est.cpu().numpy(), esto, rtol=1e-10, atol=1e-12)
    with pytest.raises(cd.CdmsError) as ei:
        cd.weights_normalize(ctx, torch.full((100,), -np.inf, dtype=torch.float64, device="cuda:0"))
        ctx.sync()
    assert ei.value.status == cd.EZEROMASS


@pytest.mark.parametrize("P", [1, 10, 257, 2048, 2049, 1_000_000])
def test_resample_bit_exact(cd, ctx, orc, P):
    import torch
    rng = np.random.default_rng(P)
    for trial in range(3):
        w = rng.exponential(size=P) * (rng.uniform(size=P) < 0.8)
        if w.sum() == 0:
            w[0] = 1.0
        if trial == 2:
            w = np.zeros(P)
            w[P // 2] = 1.0
        u = int(rng.integers(0, 2**32))
        anc = cd.resample(ctx, torch.as_tensor(w, device="cuda:0"), u)
        ctx.sync()
        st, ref = orc.resample(w, u)
        assert np.array_equal(anc.cpu().numpy(), ref)


# ---------------------------------------------------------------------------- NCCL path on one GPU
def test_nccl_one_rank_equals_local(cd, orc):
    """With a 1-rank NCCL communicator attached, every collective path (LSE all-gather, moment all-reduce,
    Q all-gather + host plan + exchange) runs; results must equal the communicator-free path bit for bit."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        ctx1 = cd.Context(0)
        ctx1.comm_init_from_torch(0, 1)
        ctx0 = cd.Context(0)
        cfg = small_cfg(J=2, K=3, ny=4, nv=4, nf=64, P=3000)
        case = Case(orc, cfg)
        xa, xb = case.dx.clone(), case.dx.clone()
        for n in range(3):
            e0, l0 = cd.bp_step(ctx0, case.scene, xa, case.dsfv, case.dy, case.m, case.v, case.eta, 0.1, 0.5, 11, n)
            e1, l1 = cd.bp_step(ctx1, case.scene, xb, case.dsfv, case.dy, case.m, case.v, case.eta, 0.1, 0.5, 11, n)
            ctx0.sync()
            ctx1.sync()
            assert torch.equal(xa, xb) and torch.equal(l0, l1)
            assert torch.allclose(e0, e1, rtol=1e-13, atol=1e-15)
        w = torch.rand(4097, dtype=torch.float64, device="cuda:0")
        a0 = cd.resample(ctx0, w, 12345)
        a1 = cd.resample(ctx1, w, 12345)
        w0, s0 = cd.weights_normalize(ctx0, torch.log(w))
        w1, s1 = cd.weights_normalize(ctx1, torch.log(w))
        ctx0.sync()
        ctx1.sync()
        assert torch.equal(a0, a1) and torch.equal(w0, w1) and torch.equal(s0, s1)
        ctx1.close()
        ctx0.close()
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- whole step
def test_bp_step_fp64_end_to_end(cd, ctx, orc):
    """c1 (10 steps): GPU bp_step in FP64 mode vs the oracle's bp_step, step by step from the same
    particles and measurements; weights (via l) within 1e-5, moments, lse, particles."""
    import torch
    cfg = scenes.CONFIGS["c1"]
    x0 = scenes.make_particles(cfg)
    xg = torch.as_tensor(x0, device="cuda:0").contiguous()
    xo = x0.copy()
    T, sv = 0.1, 0.5
    for n in range(cfg.steps):
        case = Case(orc, cfg, precision="fp64", particles=xo, step=n)
        # weights end to end: l from both sides at the predicted particles
        est, lse = cd.bp_step(ctx, case.scene, xg, case.dsfv, case.dy, case.m, case.v, case.eta, T, sv,
                              case.sc.philox_key, n)
        ctx.sync()
        st, xo, esto, lseo, anc = case.o.bp_step(xo, case.sc.sfv, case.y, case.m, case.v, case.eta, T, sv,
                                                 case.sc.philox_key, n)
        assert st == 0
        record("bp_step_particles_abs", np.max(np.abs(xg.cpu().numpy() - xo)), 1e-9, precision="fp64", step=n)
        assert abs(lse.item() - lseo) <= 1e-10 * abs(lseo)
        assert np.allclose(est.cpu().numpy(), esto, rtol=1e-8, atol=1e-10)
        assert np.allclose(xg.cpu().numpy(), xo, rtol=0, atol=1e-9), n


def test_bp_step_weights_fp64(cd, ctx, orc):
    import torch
    cfg = scenes.CONFIGS["c1"]
    case = Case(orc, cfg, precision="fp64")
    l = case.gpu_loglik(ctx)
    w, lse = cd.weights_normalize(ctx, l)
    ctx.sync()
    st, lo = case.oracle_loglik()
    st, wo, lseo = orc.normalize(lo)
    record("weights_abs", np.max(np.abs(w.cpu().numpy() - wo)), 1e-5, precision="fp64", config="c1")
    assert np.max(np.abs(w.cpu().numpy() - wo)) <= 1e-5


def test_bp_step_fp32_runs_and_is_consistent(cd, ctx, orc):
    import torch
    cfg = scenes.CONFIGS["c1"]
    case = Case(orc, cfg)
    xg = case.dx.clone()
    est, lse = cd.bp_step(ctx, case.scene, xg, case.dsfv, case.dy, case.m, case.v, case.eta, 0.1, 0.5,
                          case.sc.philox_key, 0)
    ctx.sync()
    xo = orc.predict(case.x, 0, 0.1, 0.5, case.sc.philox_key, 0)
    st, lo = case.o.loglik(xo, case.sc.sfv, case.y, case.m, case.v, case.eta)
    st, wo, lseo = orc.normalize(lo)
    assert abs(lse.item() - lseo) <= 1e-4 * max(abs(lseo), cfg.J * cfg.Nz)
    st, esto = orc.moments(xo, wo)
    assert np.allclose(est.cpu().numpy()[1:4], esto[1:4], atol=0.05)
    assert np.all(np.isfinite(xg.cpu().numpy()))


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_bp_step_fused_matches_separate(cd, orc, name):
    """The single-rank O(P) phases in one cooperative kernel (CDMS_STEP_FUSED=1, step_fused_kernel) run the same
    per-block bodies and epilogues as the five separate kernels: particles, moments and lse bit-identical."""
    import os
    cfg = scenes.CONFIGS[name]
    case = Case(orc, cfg, P=min(cfg.P, 20000))
    ctxs = []
    try:
        for f in ("0", "1"):
            os.environ["CDMS_STEP_FUSED"] = f
            ctxs.append(cd.Context(0))
    finally:
        os.environ.pop("CDMS_STEP_FUSED", None)
    outs = []
    for c in ctxs:
        xg = case.dx.clone()
        est, lse = cd.bp_step(c, case.scene, xg, case.dsfv, case.dy, case.m, case.v, case.eta, 0.1, 0.5,
                              case.sc.philox_key, 3)
        c.sync()
        outs.append((xg.cpu().numpy(), est.cpu().numpy(), lse.cpu().numpy()))
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("wf", ["spherical", "planar_wb", "planar_nb"])
def test_bp_step_graph_capture(cd, orc, wf):
    """The ABI's capture claim: after cdms_reserve ALONE (no eager warm-up call, which would allocate what reserve
    missed), one single-rank cdms_bp_step recorded in a CUDA graph on the context's stream and replayed gives
    bit-identical particles, moments and lse to an eager call made afterwards."""
    import torch
    cfg = small_cfg(J=2, K=2, ny=4, nv=4, nf=64, P=256)
    s = torch.cuda.Stream()
    ctx = cd.Context(0, s)
    case = Case(orc, cfg, wavefront=wf)
    ctx.reserve(case.scene, cfg.P)
    ctx.sync()
    key = case.sc.philox_key
    x_e, x_g = case.dx.clone(), case.dx.clone()
    est_e, lse_e = (torch.empty(28, dtype=torch.float64, device="cuda:0"),
                    torch.empty(1, dtype=torch.float64, device="cuda:0"))
    est_g, lse_g = torch.empty_like(est_e), torch.empty_like(lse_e)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        cd.bp_step(ctx, case.scene, x_g, case.dsfv, case.dy, case.m, case.v, case.eta, 0.1, 0.5, key, 0,
                   est=est_g, lse=lse_g)
    g.replay()
    ctx.sync()
    with torch.cuda.stream(s):
        cd.bp_step(ctx, case.scene, x_e, case.dsfv, case.dy, case.m, case.v, case.eta, 0.1, 0.5, key, 0,
                   est=est_e, lse=lse_e)
    ctx.sync()
    assert torch.equal(x_g, x_e) and torch.equal(est_g, est_e) and torch.equal(lse_g, lse_e)
    ctx.close()


@pytest.mark.parametrize("nf", [15, 16, 33])
@pytest.mark.parametrize("wf", ["spherical", "planar_wb"])
def test_taylor_engine_period_wrap(cd, ctx, orc, nf, wf):
    """K1T (spectral Taylor tables, taylor.cu): a 2 GHz band over few subcarriers makes df R/c span several periods,
    so the anti-periodicity sign (-1)^(N_f - 1) of the centred spectrum is exercised for odd and even N_f."""
    cfg = scenes.custom_config("wrap", J=2, K=3, ny=4, nv=4, nf=nf, P=200, fc=6.5e9, B=2e9, index=97)
    check_loglik(Case(orc, cfg, wavefront=wf), ctx, "fp32", amp=True)


def test_taylor_engine_matches_k1(cd, orc):
    """K1T and K1 (CDMS_TAYLOR=0) evaluate the same scene to within the fp32 tolerance of each other."""
    import os
    cfg = small_cfg(J=2, K=4, ny=8, nv=8, nf=128, P=300)
    ctxs = []
    try:
        ctxs.append(cd.Context(0))
        os.environ["CDMS_TAYLOR"] = "0"
        ctxs.append(cd.Context(0))
    finally:
        os.environ.pop("CDMS_TAYLOR", None)
    case = Case(orc, cfg)
    l_t = case.gpu_loglik(ctxs[0]).cpu().numpy()
    l_k = case.gpu_loglik(ctxs[1]).cpu().numpy()
    for c in ctxs:
        c.sync()
    e = rel_err(l_t, l_k, cfg.J, cfg.Nz).max()
    record("taylor_vs_k1_rel_l", e, 2e-4)
    assert e <= 2e-4, e
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("lanes", ["0", "1"])
def test_taylor_prep_fft_matches_direct(cd, orc, lanes):
    """K1T's table build by FFT (power-of-two G, tay_prep_fft_kernel) and by the direct sum (CDMS_TAY_PREP=direct)
    are both fp64 rounded once to complex64: the likelihoods agree far inside the fp32 tolerance, in both table
    layouts (CDMS_TAY_LANES)."""
    import os
    cfg = small_cfg(J=2, K=4, ny=8, nv=8, nf=64, P=500)
    ctxs = []
    try:
        os.environ["CDMS_TAY_LANES"] = lanes
        ctxs.append(cd.Context(0))
        os.environ["CDMS_TAY_PREP"] = "direct"
        ctxs.append(cd.Context(0))
    finally:
        os.environ.pop("CDMS_TAY_PREP", None)
        os.environ.pop("CDMS_TAY_LANES", None)
    case = Case(orc, cfg)
    l_f = case.gpu_loglik(ctxs[0]).cpu().numpy()
    l_d = case.gpu_loglik(ctxs[1]).cpu().numpy()
    for c in ctxs:
        c.sync()
    e = rel_err(l_f, l_d, cfg.J, cfg.Nz).max()
    record(f"taylor_fft_vs_direct_rel_l_lanes{lanes}", e, 1e-5)
    assert e <= 1e-5, e
    check_loglik(case, ctxs[0], "fp32")
    for c in ctxs:
        c.close()
