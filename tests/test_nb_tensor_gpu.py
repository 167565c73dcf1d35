"""F2: the PLANAR_NB correlation on the tensor cores (nbmma.cu) against the fp64 oracle.

In fp32, PLANAR_NB scenes run through nb_corr_kernel (tcgen05 GEMM of the delay phasors
against the snapshot) and nb_gram_kernel (closed-form Dirichlet Gram).  K1 (CDMS_NB_TENSOR=0) serves the
same scenes on the FP32 pipe.  Checked here:
  * c and G separately (cdms_loglik_terms) against the oracle's direct sums psi^H z, psi^H psi;
  * no coherent bias: mean |c| / |c_oracle| - 1 near the true position (the tensor core's fp32 accumulation
    truncates; nbmma.cu keeps the dominant product exact);
  * rel-l <= 1e-4 on shapes that exercise every tile / stage / padding edge of the GEMM;
  * agreement with K1, flags, bitwise placement independence.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2604_19723_b200 import scenes
from tests.gpu_common import Case, record, rel_err
from tests.helpers import small_cfg
from tests.test_parity_gpu import check_loglik, cd, ctx  # noqa: F401  (fixtures)

# shapes: (J, K, ny, nv, nf, P) -- UMMA N = 2 * ceil8(antennas per pass) <= 256, K stages of 32/64, ragged tiles
SHAPES = [
    dict(J=2, K=3, ny=3, nv=5, nf=100, P=77),     # N_a = 15 (padded 16), ragged stage, 308 hypotheses
    dict(J=1, K=8, ny=8, nv=8, nf=520, P=40),     # S = 9, N = 128, kc = 64, 2 accumulator pairs
    dict(J=1, K=4, ny=16, nv=16, nf=64, P=60),    # N_a = 256: two passes of N = 256, 1 accumulator pair
    dict(J=3, K=0, ny=2, nv=2, nf=300, P=65),     # S = 1
    dict(J=4, K=1, ny=1, nv=1, nf=1, P=33),       # single element, single subcarrier
    dict(J=1, K=2, ny=12, nv=10, nf=48, P=130),   # N_a = 120 -> N = 240, 3 tiles
]


def _terms_case(orc, shape, index=97):
    cfg = small_cfg(**shape, index=index)
    return cfg, Case(orc, cfg, wavefront="planar_nb", precision="fp32")


@pytest.mark.parametrize("shape", SHAPES)
def test_nb_terms_parity(cd, ctx, orc, shape):
    """c_s = psi_s^H z (tensor cores) and G = Psi^H Psi (closed form) against the oracle's direct sums."""
    cfg, case = _terms_case(orc, shape)
    l, c, G = cd.loglik_terms(ctx, case.scene, case.dx, case.dsfv, case.dy, case.m, case.v, case.eta)
    ctx.sync()
    c, G = c.cpu().numpy(), G.cpu().numpy()
    st, co, Go = case.o.terms(case.x, case.sc.sfv, case.y)
    assert st == 0
    # scale: |c| <= ||psi|| ||z|| = sqrt(Nz) ||z||; G entries <= Nz
    zn = np.sqrt(np.sum(np.abs(case.y) ** 2, axis=(1, 2)))
    ec = np.max(np.abs(c - co) / (np.sqrt(cfg.Nz) * zn[None, :, None]))
    eG = np.max(np.abs(G - Go)) / cfg.Nz
    record("nb_c_rel", ec, 1e-6, shape=shape)
    # G: closed form with fp64 set-up and range reduction, fp32 sines (nbmma.cu dirichlet_rr) -- three factors
    # of ~2 fp32 ulp each plus the carrier phasor, relative to the G scale N_z (K1's Gram terms are fp32 too)
    record("nb_G_rel", eG, 2e-6, shape=shape)
    assert ec <= 1e-6, ec
    assert eG <= 2e-6, eG


@pytest.mark.parametrize("shape", SHAPES)
def test_nb_loglik_parity(cd, ctx, orc, shape):
    cfg = small_cfg(**shape, index=97)
    check_loglik(Case(orc, cfg, wavefront="planar_nb", precision="fp32"), ctx, "fp32", amp=True)


def test_nb_pathloss_and_zero_mean(cd, ctx, orc):
    cfg = small_cfg(J=2, K=2, ny=6, nv=6, nf=64)
    check_loglik(Case(orc, cfg, wavefront="planar_nb", pathloss=True), ctx, "fp32")
    check_loglik(Case(orc, cfg, wavefront="planar_nb", mode="zm"), ctx, "fp32")


def test_nb_matches_k1(cd, orc):
    """The tensor-core path and K1 evaluate the same scene to within the fp32 tolerance of each other."""
    cfg = small_cfg(J=2, K=4, ny=8, nv=8, nf=128, P=200)
    ctxs = []
    try:
        ctxs.append(cd.Context(0))
        os.environ["CDMS_NB_TENSOR"] = "0"
        ctxs.append(cd.Context(0))
    finally:
        os.environ.pop("CDMS_NB_TENSOR", None)
    case = Case(orc, cfg, wavefront="planar_nb")
    l_tc = case.gpu_loglik(ctxs[0]).cpu().numpy()
    l_k1 = case.gpu_loglik(ctxs[1]).cpu().numpy()
    for c in ctxs:
        c.sync()
    e = rel_err(l_tc, l_k1, cfg.J, cfg.Nz).max()
    record("nb_vs_k1_rel_l", e, 2e-4)
    assert e <= 2e-4, e
    for c in ctxs:
        c.close()


def test_nb_multi_pass(cd, ctx, orc):
    """17 x 17 URA: 2 ceil8(N_a) = 592 > 256 columns -> three antenna passes (rows cut mid-row)."""
    cfg = small_cfg(J=1, K=1, ny=17, nv=17, nf=16, P=20)
    check_loglik(Case(orc, cfg, wavefront="planar_nb"), ctx, "fp32")


def test_nb_degenerate_and_invalid(cd, ctx, orc):
    import torch
    cfg = small_cfg(J=1, K=1, nf=16, P=40)
    case = Case(orc, cfg, wavefront="planar_nb")
    x = case.x.copy()
    x[7, :3] = case.sc.pa_pos[0]
    case.dx = torch.as_tensor(x, device="cuda:0").contiguous()
    l = case.gpu_loglik(ctx)
    with pytest.raises(cd.CdmsError) as ei:
        ctx.sync()
    assert ei.value.status == cd.EDEGENERATE
    l = l.cpu().numpy()
    assert l[7] == -np.inf and np.all(np.isfinite(np.delete(l, 7)))
    zero = torch.zeros_like(case.dsfv)
    cd.loglik(ctx, case.scene, case.dx, zero, case.dy, case.m, case.v, case.eta)
    with pytest.raises(cd.CdmsError) as ei:
        ctx.sync()
    assert ei.value.status == cd.EINVAL


def test_nb_near_truth_no_bias(cd, ctx, orc):
    """Particles within 1 mm of the truth: |c| is largest and the fit is most sensitive to a coherent shrink."""
    cfg = small_cfg(J=1, K=4, ny=8, nv=8, nf=256, P=32, index=97)
    rng = np.random.default_rng(5)
    x = np.zeros((32, 6))
    x[:, :3] = scenes.P_TRUE[None] + rng.uniform(-1e-3, 1e-3, size=(32, 3))
    case = Case(orc, cfg, wavefront="planar_nb", particles=x)
    _, c, _ = cd.loglik_terms(ctx, case.scene, case.dx, case.dsfv, case.dy, case.m, case.v, case.eta)
    ctx.sync()
    st, co, _ = case.o.terms(case.x, case.sc.sfv, case.y)
    c = c.cpu().numpy()
    big = np.abs(co) > 0.5 * np.abs(co).max()
    shrink = np.mean(np.abs(c[big]) / np.abs(co[big]) - 1)
    record("nb_c_shrink", abs(shrink), 2e-7)
    assert abs(shrink) <= 2e-7, shrink
    check_loglik(case, ctx, "fp32")


def test_nb_placement_independent(cd, ctx, orc):
    """Rows of the GEMM are independent: per-particle results are bitwise independent of the batch."""
    import torch
    cfg = small_cfg(J=2, K=4, ny=8, nv=8, nf=128, P=300)
    case = Case(orc, cfg, wavefront="planar_nb")
    l_full = case.gpu_loglik(ctx).cpu().numpy()
    perm = np.random.default_rng(0).permutation(cfg.P)[:123]
    sub = torch.as_tensor(case.x[perm], device="cuda:0").contiguous()
    l_sub = cd.loglik(ctx, case.scene, sub, case.dsfv, case.dy, case.m, case.v, case.eta).cpu().numpy()
    ctx.sync()
    assert np.array_equal(l_sub, l_full[perm])


def test_nb_y_scale_invariance(cd, ctx, orc):
    """y is scaled by a power of two per PA before the fp16 split: scaling z by 2^-20 scales c exactly."""
    import torch
    cfg = small_cfg(J=1, K=2, ny=4, nv=4, nf=32, P=50)
    case = Case(orc, cfg, wavefront="planar_nb")
    _, c1, _ = cd.loglik_terms(ctx, case.scene, case.dx, case.dsfv, case.dy, case.m, case.v, case.eta)
    dy2 = (case.dy * 2.0 ** -20).contiguous()
    _, c2, _ = cd.loglik_terms(ctx, case.scene, case.dx, case.dsfv, dy2, case.m, case.v, case.eta)
    ctx.sync()
    assert torch.equal(c1 * 2.0 ** -20, c2)
