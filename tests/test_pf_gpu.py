"""F1 on the GPU (cdms_pf_update): the PF-particle update message kappa~ and the PF normalization against the oracle's
orc_pf_update (itself pinned to the dense N_z x N_z definition in tests/test_oracle_pf.py) on identical inputs.

Inputs shaped like one legacy PF of the synthetic scenes: the PF is wall 1, its particles phi_p scattered around the
true SFV (+-5 cm), paired with MT particles near the true position (C-amb-8, C-amb-F1a); the other features' columns
m_l and summed mean mu3 are the scaled responses of walls 2.. at the true position (C-amb-F1b); y is the oracle's
synthetic snapshot rounded to complex64.  Tolerance: |d logr| <= 1e-4 max(|logr|, J N_z) (the rel-l reading C-amb-11;
FP32 correlations on K1T tables, fp64 assembly)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2604_19723_b200 import scenes
from tests.gpu_common import record
from tests.helpers import small_cfg


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


def _pf_inputs(orc, cfg, L, P, seed=5, wavefront="spherical"):
    sc = scenes.make_scene(cfg)
    o = orc.Oracle.from_scene(sc, wavefront=wavefront)
    y, eta = orc.measurement(o, sc, scenes.P_TRUE)
    y = y.astype(np.complex64)
    rng = np.random.default_rng(seed)
    J, Nz = cfg.J, cfg.Nz
    x = np.zeros((P, 6))
    x[:, :3] = scenes.P_TRUE + 0.01 * rng.standard_normal((P, 3))
    phi = sc.sfv[0][None, :] + 0.05 * rng.standard_normal((P, 3))
    walpha = np.full(P, 0.9 / P)
    mu = sc.rho[1] * (1 + 0.1 * (rng.standard_normal(P) + 1j * rng.standard_normal(P)))
    gamma = np.full(P, 0.02)
    zeta = np.full(J, 0.9)
    mcols = np.zeros((J, L, Nz), dtype=np.complex128)
    mu3 = np.zeros((J, Nz), dtype=np.complex128)
    for j in range(J):
        for l in range(L):
            st, psi = o.response(scenes.P_TRUE, j, 2 + l, sc.sfv)
            assert st == 0
            mcols[j, l] = np.sqrt(0.05) * psi
            mu3[j] += 0.9 * sc.rho[2 + l] * psi
    mcols = mcols.astype(np.complex64)
    mu3 = mu3.astype(np.complex64)
    return sc, o, y, np.full(J, eta), x, phi, walpha, mu, gamma, zeta, mu3, mcols


@pytest.mark.parametrize("name,L,P,los", [("c2", 0, 300, False), ("c2", 3, 300, False), ("c3", 5, 120, False),
                                           ("c4", 3, 64, False), ("c5", 7, 40, False), ("c2", 3, 300, True),
                                           ("c3", 5, 120, True)])
@pytest.mark.parametrize("wavefront", ["spherical", "planar_wb"])
def test_pf_update_parity(cd, ctx, orc, name, L, P, los, wavefront):
    """los: the LOS PF s = 0 (d_phi = NULL; the F4 driver's slot 0)."""
    import torch
    base = scenes.CONFIGS[name]
    cfg = small_cfg(J=base.J, K=max(base.K, L + 1), ny=base.ny, nv=base.nv, nf=base.nf, P=P, index=base.index)
    sc, o, y, eta, x, phi, wa, mu, gamma, zeta, mu3, mcols = _pf_inputs(orc, cfg, L, P, wavefront=wavefront)
    scene = cd.Scene.from_synthetic(sc, wavefront=wavefront)
    dev = "cuda:0"
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
    logr, w, out = cd.pf_update(ctx, scene, t(x), None if los else t(phi), t(wa), t(mu.astype(np.complex128)),
                                t(gamma), zeta, eta, t(y), t(mu3), t(mcols) if L else None)
    ctx.sync()
    st, lo, wo, logMo, exo = o.pf_update(x, None if los else phi, wa, mu, gamma, zeta, eta, y.astype(np.complex128),
                                         mu3.astype(np.complex128), mcols.astype(np.complex128))
    assert st == 0
    lg = logr.cpu().numpy()
    e = np.abs(lg - lo) / np.maximum(np.abs(lo), cfg.J * cfg.Nz)
    record("pf_logr_rel", e.max(), 1e-4, config=name, L=L, wavefront=wavefront, los=los)
    assert e.max() <= 1e-4, e.max()
    # the kernel's own normalization (S-IV) is consistent with its logr
    logM, ex = out.cpu().numpy()
    wg = w.cpu().numpy()
    assert np.allclose(wg, np.exp(lg - logM), rtol=1e-12)
    assert abs(wg.sum() + (1 - wa.sum()) * np.exp(-logM) - 1.0) < 1e-10 and 0.0 <= ex <= 1.0 + 1e-12
    # and equals the oracle's normalization of the same logr
    mx = max(lg.max(), 0.0)
    logM_ref = mx + np.log(np.exp(lg - mx).sum() + (1 - wa.sum()) * np.exp(-mx))
    assert abs(logM - logM_ref) <= 1e-10 * max(1.0, abs(logM_ref))


def test_pf_update_null_feature_and_errors(cd, ctx, orc):
    """q = mu = 0: every log-ratio is log w_alpha and the existence stays the prior sum (as the oracle pin)."""
    import torch
    cfg = small_cfg(J=2, K=3, ny=4, nv=4, nf=64, P=50, index=2)
    sc, o, y, eta, x, phi, wa, mu, gamma, zeta, mu3, mcols = _pf_inputs(orc, cfg, 2, 50)
    scene = cd.Scene.from_synthetic(sc)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda:0")  # noqa: E731
    logr, w, out = cd.pf_update(ctx, scene, t(x), t(phi), t(wa), t(0 * mu.astype(np.complex128)), t(0 * gamma), zeta,
                                eta, t(y), t(mu3), t(mcols))
    ctx.sync()
    assert np.allclose(logr.cpu().numpy(), np.log(wa), atol=1e-12, rtol=0)
    assert abs(out[1].item() - wa.sum()) < 1e-12
    bad = cd.Scene.from_synthetic(sc, precision="fp64")
    with pytest.raises(cd.CdmsError) as ei:
        cd.pf_update(ctx, bad, t(x), t(phi), t(wa), t(mu.astype(np.complex128)), t(gamma), zeta, eta, t(y), t(mu3),
                     t(mcols))
    assert ei.value.status == cd.EUNSUPPORTED
