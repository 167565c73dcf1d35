"""F4 update messages on the GPU against the oracle (tests/test_oracle_noise_ppr.py pins the oracle to the dense
definitions): the noise variance update nu~ with the normalized noise weights (cdms_noise_update, P:L1057-1126,
P:L3398-3410) and the PPR update omega~ with the existence sigma(u) (cdms_ppr_update, S-VI).

Inputs shaped like the synthetic scenes: y the oracle's snapshot (complex64), the features' columns = sqrt(0.05) x their
responses at the true position, mu_nu = 0.9 sum_s rho_s psi_s, noise particles eta_p = eta_true x Gamma(10)/10 (the
Gamma transition of P:L3783-3784 around the true level), w_xi uniform.  Both sides read the same complex64 vectors and
form their N_z-long dot products in fp64, so the results agree to ~1e-12 relative (GPU: eigendecomposition of M^H M
once per PA; oracle: the paper's per-particle Cholesky)."""
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


def _inputs(orc, name, S):
    base = scenes.CONFIGS[name]
    cfg = small_cfg(J=base.J, K=max(base.K, S - 1), ny=base.ny, nv=base.nv, nf=base.nf, P=64, index=base.index)
    sc = scenes.make_scene(cfg)
    o = orc.Oracle.from_scene(sc)
    y, eta = orc.measurement(o, sc, scenes.P_TRUE)
    J, Nz = cfg.J, cfg.Nz
    cols = np.zeros((J, S, Nz), dtype=np.complex128)
    mu = np.zeros((J, Nz), dtype=np.complex128)
    for j in range(J):
        for s in range(S):
            st, psi = o.response(scenes.P_TRUE, j, s, sc.sfv)
            cols[j, s] = np.sqrt(0.05) * psi
            mu[j] += 0.9 * sc.rho[s] * psi
    c64 = lambda a: a.astype(np.complex64)  # noqa: E731
    return cfg, sc, o, c64(y.reshape(J, -1)), eta, c64(mu), c64(cols)


@pytest.mark.parametrize("name,S", [("c2", 5), ("c3", 7), ("c5", 9), ("c2", 0)])
def test_noise_update_parity(cd, ctx, orc, name, S):
    import torch
    cfg, sc, o, y, eta, mu, cols = _inputs(orc, name, S)
    rng = np.random.default_rng(1)
    P = 5000
    etas = eta * rng.gamma(10.0, 0.1, (cfg.J, P))
    wxi = np.full((cfg.J, P), 1.0 / P)
    scene = cd.Scene.from_synthetic(sc)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda:0")  # noqa: E731
    shp = (cfg.J, cfg.nf, cfg.Na)
    logw, w, ln = cd.noise_update(ctx, scene, t(etas), t(wxi), t(y.reshape(shp)), t(mu.reshape(shp)),
                                  t(cols.reshape(cfg.J, S, cfg.nf, cfg.Na)) if S else None)
    ctx.sync()
    st, lo, wo, lno = o.noise_update(etas, wxi, y.astype(np.complex128), mu.astype(np.complex128),
                                     cols.astype(np.complex128))
    assert st == 0
    e = np.max(np.abs(logw.cpu().numpy() - lo) / np.maximum(1.0, np.abs(lo)))
    ew = np.max(np.abs(w.cpu().numpy() - wo))
    # both sides sum N_z-long fp64 dot products (relative error ~sqrt(N_z) 1e-16) into |e|^2/eta and the Woodbury term,
    # which cancel by up to ~1e4 into log nu~: 1e-9 relative bounds that floor at N_z = 65536 (measured 2.6e-10 at c5)
    record("noise_logw_rel", e, 1e-9, config=name, S=S)
    record("noise_w_abs", ew, 1e-8, config=name, S=S)
    assert e <= 1e-9, e
    assert ew <= 1e-8, ew
    assert np.allclose(ln.cpu().numpy(), lno, rtol=1e-12)


@pytest.mark.parametrize("name,L", [("c2", 3), ("c3", 5), ("c5", 7), ("c2", 0)])
def test_ppr_update_parity(cd, ctx, orc, name, L):
    import torch
    cfg, sc, o, y, eta, mu3, cols = _inputs(orc, name, L + 2)
    J, Nz = cfg.J, cfg.Nz
    # the PF s = the last wall: its ray m_omega and mean mu4 from its response at the truth; the other L features as M
    momega, mu4 = np.sqrt(0.05) * cols[:, -1] / np.sqrt(0.05), np.zeros((J, Nz), dtype=np.complex64)
    momega = (np.sqrt(0.1) * momega).astype(np.complex64)
    mu4 = (0.5 * cols[:, -1] / np.sqrt(0.05)).astype(np.complex64)
    mcols = cols[:, :L]
    zeta = np.full(J, 0.3)
    etas = np.full(J, eta)
    scene = cd.Scene.from_synthetic(sc)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda:0")  # noqa: E731
    shp = (J, cfg.nf, cfg.Na)
    out = cd.ppr_update(ctx, scene, zeta, etas, t(y.reshape(shp)), t(mu3.reshape(shp)), t(momega.reshape(shp)),
                        t(mu4.reshape(shp)), t(mcols.reshape(J, L, cfg.nf, cfg.Na)) if L else None)
    ctx.sync()
    st, oo = o.ppr_update(zeta, etas, y.astype(np.complex128), mu3.astype(np.complex128),
                          mcols.astype(np.complex128), momega.astype(np.complex128), mu4.astype(np.complex128))
    assert st == 0
    og = out.cpu().numpy()
    e = np.max(np.abs(og[:, :2] - oo[:, :2]) / np.maximum(1.0, np.abs(oo[:, :2])))
    record("ppr_logratio_rel", e, 1e-10, config=name, L=L)
    assert e <= 1e-10, e
    assert np.max(np.abs(og[:, 2] - oo[:, 2])) <= 1e-10
