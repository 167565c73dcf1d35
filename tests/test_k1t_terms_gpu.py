"""Element-level parity of the default FP32 engine K1T (taylor.cu: spectral Taylor tables for c, closed-form Gram for
G), in both table layouts / correlation kernels (lane groups [g][h][m], thread per particle [m][g][l]):

* per response element (north_star: |d phase| <= 1e-4 rad): with a one-hot snapshot y = delta(k, m) the
  kernel's correlation is c_s = psi_s^H y = conj(psi_s[k, m]), so cdms_loglik_terms exposes K1T's own
  value of every sampled response element -- its set-up (tay_locate, TwoSum, magic-constant rounding), its tables and
  its Taylor evaluation -- for comparison with the oracle's element-by-element fp64 response;
* c = Psi^H z and G = Psi^H Psi element by element against the oracle's direct sums (orc_terms), with particles placed
  at controlled distances from a wall plane, where the LOS and that wall's component have (nearly) equal delays and
  the Gram's Dirichlet factor D_N(x) is evaluated at |x| from 0 through its small-argument branch (P:L769 fn,
  P:L1016-1022, reading C-amb-13).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2604_19723_b200 import scenes
from tests.gpu_common import Case, record
from tests.helpers import small_cfg

SHAPES = {  # the BASELINE configs' scene shapes (J, K, URA, N_f)
    "c2": dict(J=1, K=4, ny=8, nv=8, nf=128),
    "c3": dict(J=2, K=6, ny=8, nv=8, nf=512),
    "c4": dict(J=1, K=4, ny=16, nv=16, nf=256),
    "c5": dict(J=4, K=8, ny=8, nv=8, nf=1024),
    # more than 64 antennas per lane: the Gram's chunked path (fp32 sums of 16 antennas, fp64 totals in shared
    # memory; S = 9 in two pair parts) instead of the single-pass one every BASELINE config but c4 takes
    "s9a144": dict(J=1, K=8, ny=12, nv=12, nf=64),
    "s7a144": dict(J=1, K=6, ny=12, nv=12, nf=128),
    # J N_a,pad > 512: the correlation kernel reads its template columns from global memory, not the constant bank
    "j4a144": dict(J=4, K=2, ny=12, nv=12, nf=64),
    # a 2 GHz band (c/df = 9.6 m): component paths differ by more than half a delay period, so the S = 9 Gram's W0
    # kernel flags the batch and its fallback recomputes it; the correlation takes the TwoSum locate
    "s9wide": dict(J=1, K=8, ny=8, nv=8, nf=64, B=2e9),
}
LAYOUTS = {"lanes": "1", "thread": "0"}


@pytest.fixture(scope="module")
def cd():
    from paper_2604_19723_b200 import build as B
    B.build()
    from paper_2604_19723_b200 import cdms
    return cdms


@pytest.fixture(scope="module")
def ctxs(cd):
    out = {}
    try:
        for name, v in LAYOUTS.items():
            os.environ["CDMS_TAY_LANES"] = v
            out[name] = cd.Context(0)
    finally:
        os.environ.pop("CDMS_TAY_LANES", None)
    yield out
    for c in out.values():
        c.close()


def _particles(cfg, n, seed):
    rng = np.random.default_rng(seed)
    x = np.zeros((n, 6))
    x[:, :3] = scenes.ROI_LO + (scenes.ROI_HI - scenes.ROI_LO) * rng.uniform(size=(n, 3))
    x[: n // 4, :3] = scenes.P_TRUE + rng.uniform(-1e-3, 1e-3, size=(n // 4, 3))
    return x


@pytest.mark.parametrize("wf", ["spherical", "planar_wb"])
@pytest.mark.parametrize("layout", list(LAYOUTS))
@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_k1t_element_phase_onehot(cd, ctxs, orc, name, layout, wf):
    import torch
    ctx = ctxs[layout]
    shp = SHAPES[name]
    cfg = small_cfg(**shp, P=12, index=4 if name == "c5" else 2)
    sc = scenes.make_scene(cfg)
    o = orc.Oracle.from_scene(sc, wavefront=wf)
    scene = cd.Scene.from_synthetic(sc, wavefront=wf)
    x = _particles(cfg, cfg.P, 5)
    dx = torch.as_tensor(x, device="cuda:0").contiguous()
    dsfv = torch.as_tensor(sc.sfv, device="cuda:0").contiguous()
    m = np.zeros((cfg.J, cfg.S), dtype=complex)
    v = np.full((cfg.J, cfg.S), 0.1)
    eta = np.ones(cfg.J)
    rng = np.random.default_rng(11)
    ks = [0, cfg.nf - 1] + list(rng.integers(0, cfg.nf, 6))
    ms = [0, cfg.Na - 1] + list(rng.integers(0, cfg.Na, 6))
    # oracle responses of every (particle, PA, component): only the sampled elements are kept
    n_idx = [k * cfg.Na + mm for k, mm in zip(ks, ms)]
    ref = np.zeros((cfg.P, cfg.J, cfg.S, len(n_idx)), dtype=complex)
    for p in range(cfg.P):
        for j in range(cfg.J):
            for s in range(cfg.S):
                st, psi = o.response(x[p, :3], j, s, sc.sfv)
                assert st == 0
                ref[p, j, s] = psi[n_idx]
    worst_ph, worst_mag = 0.0, 0.0
    for e, (k, mm) in enumerate(zip(ks, ms)):
        y = np.zeros((cfg.J, cfg.nf, cfg.Na), dtype=np.complex64)
        y[:, k, mm] = 1.0
        l, c, G = cd.loglik_terms(ctx, scene, dx, dsfv, torch.as_tensor(y, device="cuda:0"), m, v, eta)
        ctx.sync()
        psi_gpu = np.conj(c.cpu().numpy())            # c_s = conj(psi_s[k, m]) for the one-hot snapshot
        worst_ph = max(worst_ph, float(np.max(np.abs(np.angle(psi_gpu * np.conj(ref[..., e]))))))
        worst_mag = max(worst_mag, float(np.max(np.abs(np.abs(psi_gpu) - 1.0))))
    record("k1t_phase_rad", worst_ph, 1e-4, config=name, layout=layout, wavefront=wf)
    record("k1t_magnitude", worst_mag, 1e-4, config=name, layout=layout, wavefront=wf)
    assert worst_ph <= 1e-4, worst_ph
    assert worst_mag <= 1e-4, worst_mag


def _equal_delay_particles(cfg, sc, rng, n):
    """Particles at distance delta from the plane of wall 1 (inside the room), delta log-uniform in [1e-7, 0.1] m
    plus delta = 0: the LOS and the wall-1 component then differ in delay by ~2 delta cos(theta) (equal on the
    plane, where the mirror symmetry makes every antenna's distances equal too)."""
    s = sc.sfv[0]
    nrm = s / np.linalg.norm(s)
    a = np.linalg.norm(s) / 2.0                      # wall {x : n.x = a}
    x = np.zeros((n, 6))
    delta = np.concatenate([[0.0], 10.0 ** rng.uniform(-7, -1, n - 1)])
    base = scenes.ROI_LO + (scenes.ROI_HI - scenes.ROI_LO) * rng.uniform(size=(n, 3))
    x[:, :3] = base - (base @ nrm - a + delta)[:, None] * nrm[None, :]
    return x, delta


@pytest.mark.parametrize("wf", ["spherical", "planar_wb"])
@pytest.mark.parametrize("layout", list(LAYOUTS))
@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5", "s9a144", "s7a144", "j4a144", "s9wide"])
def test_k1t_terms_parity(cd, ctxs, orc, name, layout, wf):
    """c and G of K1T against orc_terms (direct sums over the element-wise fp64 responses), ROI particles and
    equal-delay particles near a wall plane; spherical and planar wideband responses."""
    import torch
    ctx = ctxs[layout]
    shp = SHAPES[name]
    cfg = small_cfg(**shp, P=48, index=4 if name == "c5" else 2)
    case = Case(orc, cfg, particles=np.zeros((1, 6)), wavefront=wf)
    rng = np.random.default_rng(7)
    xe, delta = _equal_delay_particles(cfg, case.sc, rng, 32)
    x = np.concatenate([_particles(cfg, 16, 3), xe])
    dx = torch.as_tensor(x, device="cuda:0").contiguous()
    l, c, G = cd.loglik_terms(ctx, case.scene, dx, case.dsfv, case.dy, case.m, case.v, case.eta)
    ctx.sync()
    c, G = c.cpu().numpy(), G.cpu().numpy()
    st, co, Go = case.o.terms(x, case.sc.sfv, case.y)
    assert st == 0
    zn = np.sqrt(np.sum(np.abs(case.y) ** 2, axis=(1, 2)))
    ec = np.abs(c - co) / (np.sqrt(cfg.Nz) * zn[None, :, None])
    eG = np.abs(G - Go) / cfg.Nz
    # G_01 of the equal-delay particles (LOS vs wall 1) against its delay offset
    worst = int(np.argmax(eG.max(axis=(1, 2, 3))))
    record("k1t_c_rel", ec.max(), 1e-6, config=name, layout=layout, wavefront=wf)
    record("k1t_G_rel", eG.max(), 2e-6, config=name, layout=layout, wavefront=wf,
           worst_particle=worst, worst_delta=float(delta[worst - 16]) if worst >= 16 else None)
    assert ec.max() <= 1e-6, ec.max()
    assert eG.max() <= 2e-6, (eG.max(), worst, delta[worst - 16] if worst >= 16 else None)
    assert np.allclose(np.real(np.einsum("pjss->pjs", G)), cfg.Nz, rtol=1e-12)   # G_ss = N_z (unit modulus)


@pytest.mark.parametrize("name", ["c5", "c3"])
def test_k1t_terms_sampled_at_bench_launch(cd, orc, name):
    """c and G at the launch configuration the bench times for these shapes: P J >= 2 x 148 x 1024 threads, so the Gram
    runs one lane per particle (lsplit 0) and, at S = 9, all 36 pairs in one part; the correlation is the
    thread-per-particle kernel.  The oracle computes 24 sampled particles (first, last, random) one by one."""
    import torch
    shp = SHAPES[name]
    P = -(-2 * 148 * 1024 // shp["J"]) + 1000
    cfg = small_cfg(**shp, P=P, index=4 if name == "c5" else 2)
    case = Case(orc, cfg, particles=np.zeros((1, 6)), wavefront="spherical")
    x = _particles(cfg, P, 13)
    ctx = cd.Context(0)
    dx = torch.as_tensor(x, device="cuda:0").contiguous()
    l, c, G = cd.loglik_terms(ctx, case.scene, dx, case.dsfv, case.dy, case.m, case.v, case.eta)
    ctx.sync()
    rng = np.random.default_rng(17)
    idx = np.unique(np.concatenate([[0, P - 1], rng.integers(0, P, 22)]))
    ti = torch.as_tensor(idx, device="cuda:0")
    c, G = c.index_select(0, ti).cpu().numpy(), G.index_select(0, ti).cpu().numpy()
    ctx.close()
    st, co, Go = case.o.terms(x[idx], case.sc.sfv, case.y)
    assert st == 0
    zn = np.sqrt(np.sum(np.abs(case.y) ** 2, axis=(1, 2)))
    ec = np.abs(c - co) / (np.sqrt(cfg.Nz) * zn[None, :, None])
    eG = np.abs(G - Go) / cfg.Nz
    record("k1t_c_rel_bench_launch", ec.max(), 1e-6, config=name, P=P)
    record("k1t_G_rel_bench_launch", eG.max(), 2e-6, config=name, P=P)
    assert ec.max() <= 1e-6, ec.max()
    assert eG.max() <= 2e-6, eG.max()


@pytest.mark.parametrize("sfv_pp", [False, True])
def test_locality_order_is_bit_identical(cd, orc, sfv_pp):
    """With CDMS_LOCALITY=1, batches from 32768 particles run in Morton order (sort.cu) and the assembly writes every
    result back to its particle: l and the LMMSE amplitudes must equal the default (unsorted) evaluation bit for bit."""
    import torch
    cfg = small_cfg(**SHAPES["c2"], P=70000, index=2)
    case = Case(orc, cfg, particles=scenes.make_particles(scenes.CONFIGS["c2"], 0, 70000))
    ctxs = []
    try:
        ctxs.append(cd.Context(0))
        os.environ["CDMS_LOCALITY"] = "1"
        ctxs.append(cd.Context(0))
    finally:
        os.environ.pop("CDMS_LOCALITY", None)
    sfv = case.dsfv
    if sfv_pp:
        rng = np.random.default_rng(9)
        s = case.sc.sfv[None] * (1.0 + 0.01 * rng.standard_normal((cfg.P, cfg.K, 3)))
        sfv = torch.as_tensor(s, device="cuda:0").contiguous()
    outs = []
    for c in ctxs:
        l, a = cd.loglik(c, case.scene, case.dx, sfv, case.dy, case.m, case.v, case.eta, sfv_per_particle=sfv_pp,
                         want_amp=True)
        c.sync()
        outs.append((l.cpu().numpy(), a.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    for c in ctxs:
        c.close()
