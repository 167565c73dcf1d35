"""F4 on the GPU: one step of the SLAM driver (cdms_slam_step) against the oracle's step (oracle/slam.py, pinned in
tests/test_oracle_slam.py) from the same state, the same complex64 snapshot and the same Philox counters.

State: a known scene (LOS and the true walls as PFs at the true SFVs and amplitudes, MT particles within 1 mm of the
truth) plus a PF at a wrong SFV, so one step exercises every message, a birth, declaration and pruning.  The MT
likelihood runs in FP64 (K1), the PF updates in FP32 on K1T tables (their only engine), everything else in fp64.

Tolerances: transitions and belief sums 1e-9 relative (fp64 on both sides, different summation orders; the birth slot
inherits the F3 proposal's ~1e-7 agreement); MT log-likelihood 1e-8 relative (the FP64 engine's bar); PF log-ratios
1e-4 max(|logr|, J N_z) (the F1 bar, FP32 correlations); PPR log ratios 1e-5 and noise weights 1e-7
(complex64 columns); estimates 1e-6 (weights from l)."""
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


def _known_state(OS, cfg, sc, P, eta, weak=True):
    rng = np.random.default_rng(0)
    x = np.zeros((P, 6))
    x[:, :3] = scenes.P_TRUE + 0.001 * rng.standard_normal((P, 3))
    x[:, 3:] = 0.1 * rng.standard_normal((P, 3))
    full = lambda v: np.full(P, v)  # noqa: E731
    slots = [OS.Slot(None, full(sc.rho[0]) * (1 + 0.01 * rng.standard_normal(P)), full(1e-3), full(1.0 / P),
                     np.full(cfg.J, 0.9), 0)]
    for k in range(cfg.K):
        phi = sc.sfv[k][None, :] + 0.002 * rng.standard_normal((P, 3))
        slots.append(OS.Slot(phi, full(sc.rho[k + 1]), full(1e-3), full(0.95 / P), np.full(cfg.J, 0.8), k + 1))
    if weak:
        slots.append(OS.Slot(np.tile([30.0, 30.0, 0.0], (P, 1)), full(1e-4 + 0j), full(1e-4), full(0.02 / P),
                             np.full(cfg.J, 0.5), cfg.K + 1))
    phi_hat = {s.ident: (np.mean(s.phi, axis=0) if s.phi is not None else None) for s in slots}
    eta0 = eta * (1.0 + 0.2 * rng.uniform(-1, 1, (cfg.J, P)))
    return OS.State(x, eta0, slots, n=1, next_id=len(slots), phi_hat=phi_hat)


def _load(cd, slam, st, torch):
    v = slam.view()
    v["x"].copy_(torch.as_tensor(st.x))
    v["eta"].copy_(torch.as_tensor(st.eta))
    for i, s in enumerate(st.slots):
        if s.phi is not None:
            v["phi"][i].copy_(torch.as_tensor(s.phi))
        v["mu"][i].copy_(torch.as_tensor(s.mu.astype(np.complex128)))
        v["gamma"][i].copy_(torch.as_tensor(s.gamma))
        v["w"][i].copy_(torch.as_tensor(s.w))
    S = len(st.slots)
    zeta = np.stack([s.zeta for s in st.slots])
    ph = np.stack([st.phi_hat[s.ident] if s.phi is not None else np.zeros(3) for s in st.slots])
    slam.set_slots([s.ident for s in st.slots], zeta, ph, n=st.n, next_id=st.next_id)
    assert slam.view()["n_slots"] == S


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("J,K,nf,wf", [(2, 2, 16, "spherical"), (1, 3, 32, "spherical"), (2, 2, 16, "planar_wb")])
def test_slam_step_matches_oracle(cd, ctx, orc, J, K, nf, wf):
    import torch
    from oracle import slam as OS
    cfg = small_cfg(J=J, K=K, ny=4, nv=4, nf=nf, P=64, index=5)
    sc = scenes.make_scene(cfg)
    base = orc.Oracle.from_scene(sc, wavefront=wf)
    y, eta = orc.measurement(base, sc, scenes.P_TRUE)
    y64 = y.astype(np.complex64)
    P = 256
    prm = OS.Params(P_m=64, N_g=512)
    st = _known_state(OS, cfg, sc, P, eta)
    scene = cd.Scene.from_synthetic(sc, wavefront=wf, precision="fp64")
    slam = cd.Slam(ctx, scene, P, P_m=prm.P_m, N_g=prm.N_g, key=prm.key, keep_debug=1)
    _load(cd, slam, st, torch)
    rep = slam.step(torch.as_tensor(y64, device="cuda:0"))
    ctx.sync()
    v = slam.view()
    new, ref = OS.step(base, st, y64.astype(np.complex128), prm)
    S = ref["n_slots"]
    assert rep["n_feat"] == S
    # (i) prediction messages and the birth
    e_x = float(np.max(np.abs(v["x_pred"].cpu().numpy() - ref["x_pred"])))
    e_eta = _rel(v["eta_pred"].cpu().numpy(), ref["eta_pred"])
    record("slam_x_pred_abs", e_x, 1e-12, J=J, K=K, wavefront=wf)
    record("slam_eta_pred_rel", e_eta, 1e-12, J=J, K=K)
    assert e_x <= 1e-12 and e_eta <= 1e-12
    for i, s in enumerate(ref["slots_prior"]):
        tol = 1e-6 if i == S - 1 and S > len(st.slots) else 1e-12       # the birth: F3's mu_q, C_q to ~1e-7
        if s.phi is not None:
            assert _rel(v["phi_prior"][i].cpu().numpy(), s.phi) <= tol, i
        assert _rel(v["mu_prior"][i].cpu().numpy(), s.mu) <= tol, i
        assert _rel(v["gamma_prior"][i].cpu().numpy(), s.gamma) <= tol, i
        assert _rel(v["w_prior"][i].cpu().numpy(), s.w) <= max(tol, 1e-12), i
    assert np.allclose(rep["x_pred_hat"], ref["x_pred_hat"], rtol=0, atol=1e-12)
    assert np.allclose(rep["eta_bar"], ref["eta_bar"], rtol=1e-12)
    # belief-averaged columns (reading F4c)
    born = S > len(st.slots)
    eb, ebb = 0.0, 0.0
    for name, key in (("u_sums", "u"), ("m_sums", "m"), ("mw_sums", "momega")):
        g = v[name].cpu().numpy()[:, :S]
        o = ref[key]
        for s in range(S):
            e = _rel(g[:, s], o[:, s]) if np.max(np.abs(o[:, s])) > 0 else float(np.max(np.abs(g[:, s])))
            if born and s == S - 1:
                ebb = max(ebb, e)
            else:
                eb = max(eb, e)
    # legacy slots: fp64 on identical particles; the birth slot's particles inherit the F3 proposal's (mu_q, C_q)
    # agreement (~1e-7 relative, tests/test_birth_gpu.py), i.e. SFV offsets of ~1e-6 m: phases of 2 pi 1e-6 / lambda
    record("slam_belief_cols_rel", eb, 1e-9, J=J, K=K)
    record("slam_belief_cols_birth_rel", ebb, 1e-4, J=J, K=K)
    assert eb <= 1e-9, eb
    assert ebb <= 1e-4, ebb
    # iota~ (FP64), nu~, kappa~ (FP32), omega~
    l_g, l_o = v["loglik"].cpu().numpy(), ref["l"]
    e_l = float(np.max(np.abs(l_g - l_o) / np.maximum(np.abs(l_o), 1.0)))
    record("slam_loglik_rel", e_l, 1e-8, J=J, K=K)
    assert e_l <= 1e-8, e_l
    # nu~ reads mu_nu and the columns in complex64 (the ABI's vector type) where the oracle keeps fp64
    e_we = float(np.max(np.abs(v["w_eta"].cpu().numpy() - ref["w_eta"])))
    record("slam_w_eta_abs", e_we, 1e-7, J=J, K=K)
    assert e_we <= 1e-7, e_we
    Nz = cfg.Nz
    lg = v["logr"].cpu().numpy()
    pf_g = v["pf_out"].cpu().numpy()
    ppr_g = v["ppr_out"].cpu().numpy()
    e_pf, e_pr, e_ex = 0.0, 0.0, 0.0
    for s in range(S):
        logr_o, logM_o, ex_o = ref["pf"][s]
        fin = np.isfinite(logr_o)
        e_pf = max(e_pf, float(np.max(np.abs(lg[s][fin] - logr_o[fin]) / np.maximum(np.abs(logr_o[fin]), J * Nz))))
        e_ex = max(e_ex, abs(pf_g[s, 1] - ex_o))
        o = ref["ppr"][s]
        e_pr = max(e_pr, float(np.max(np.abs(ppr_g[s, :J, :2] - o[:, :2]) / np.maximum(1.0, np.abs(o[:, :2])))))
    record("slam_pf_logr_rel", e_pf, 1e-4, J=J, K=K)
    record("slam_exist_abs", e_ex, 0.05, J=J, K=K)
    # omega~: the driver hands the columns to cdms_ppr_update in complex64 (the ABI's vector type, 6e-8 relative) while
    # the oracle keeps fp64; |e|^2/eta-sized terms cancel into the log ratio, so 1e-5 relative to max(1, |ratio|)
    record("slam_ppr_rel", e_pr, 1e-5, J=J, K=K)
    assert e_pf <= 1e-4, e_pf
    assert e_ex <= 0.05, e_ex
    assert e_pr <= 1e-5, e_pr
    # estimates, declaration, pruning, the next state
    # the MT weights come from l (1e-8 relative: |d l| up to ~1e-8 |l| nats), so the weighted moments agree to ~1e-6
    e_est = float(np.max(np.abs(rep["est"] - ref["est"]) / np.maximum(np.abs(ref["est"]), 1e-3)))  # >= 1 mm scale
    record("slam_est_rel", e_est, 1e-6, J=J, K=K)
    assert e_est <= 1e-6, e_est
    assert np.allclose(rep["eta_hat"], ref["eta_hat"], rtol=1e-8)
    feats = ref["features"]
    assert rep["ident"] == [f["ident"] for f in feats]
    assert rep["declared"] == [f["declared"] for f in feats]
    assert [i for i, p in zip(rep["ident"], rep["pruned"]) if not p] == [s.ident for s in new.slots]
    for i, f in enumerate(feats):
        if f["phi"] is not None and f["exist"] > 1e-6:
            # PF weights from FP32 log-ratios: the weighted mean moves by a small fraction of the 2 mm spread
            assert np.allclose(rep["phi_hat"][i], f["phi"], rtol=0, atol=1e-5)
        assert np.allclose(rep["zeta"][i], f["zeta"], rtol=0, atol=1e-5)   # sigma(u), u within the PPR bar
    xg = v["x"].cpu().numpy()
    # rows equal up to the regularization's Cholesky factor (covariance from weights within ~1e-6): 1 um, while a
    # different ancestor is ~1 mm away
    same = np.mean(np.all(np.abs(xg - new.x) <= 1e-6, axis=1))
    # resampling quantizes e^{l - M} at 2^-36 (C-amb-23): l within 1e-8 relative moves a few slot boundaries of 256
    record("slam_mt_rows_equal", same, 0.95, J=J, K=K)
    assert same >= 0.95, same
    slam.close()


def test_slam_init_and_multistep_runs(cd, ctx, orc):
    """cdms_slam_init (the LOS alone) and a few steps: births up to the slot limit, every report valid."""
    import torch
    cfg = small_cfg(J=2, K=2, ny=4, nv=4, nf=16, P=64, index=5)
    sc = scenes.make_scene(cfg)
    base = orc.Oracle.from_scene(sc)
    y, eta = orc.measurement(base, sc, scenes.P_TRUE)
    P = 2048
    scene = cd.Scene.from_synthetic(sc)
    slam = cd.Slam(ctx, scene, P, P_m=128, N_g=1024)
    rng = np.random.default_rng(3)
    x0 = np.zeros((P, 6))
    x0[:, :3] = scenes.P_TRUE + 0.01 * rng.standard_normal((P, 3))
    slam.init(torch.as_tensor(x0, device="cuda:0"), torch.full((cfg.J, P), eta, dtype=torch.float64, device="cuda:0"))
    dy = torch.as_tensor(y.astype(np.complex64), device="cuda:0")
    for k in range(4):
        r = slam.step(dy)
        assert r["n"] == k + 1 and r["ident"][0] == 0 and not r["pruned"][0]
        assert np.all((r["exist"] >= 0) & (r["exist"] <= 1 + 1e-9))
        assert np.all(np.isfinite(r["est"])) and np.all(r["eta_hat"] > 0)
        assert 1 <= r["n_slots"] <= r["n_feat"] <= 9
    ctx.sync()
    slam.close()


def test_slam_full_slots_and_empty_box(cd, ctx, orc):
    """Edge cases of the driver against the oracle: all 9 slots taken (no birth, P:L3257 Q = 1 needs a free slot) and a
    snapshot without power (the proposal fails with no residual: no birth); the oracle's step makes the same
    decisions."""
    import torch
    from oracle import slam as OS
    cfg = small_cfg(J=1, K=8, ny=4, nv=4, nf=16, P=64, index=5)
    sc = scenes.make_scene(cfg)
    base = orc.Oracle.from_scene(sc)
    y, eta = orc.measurement(base, sc, scenes.P_TRUE)
    y64 = y.astype(np.complex64)
    P = 128
    # (a) 9 slots: LOS + 8 walls
    prm = OS.Params(P_m=32, N_g=256)
    st = _known_state(OS, cfg, sc, P, eta, weak=False)
    assert len(st.slots) == 9
    scene = cd.Scene.from_synthetic(sc, precision="fp64")
    slam = cd.Slam(ctx, scene, P, P_m=prm.P_m, N_g=prm.N_g, key=prm.key, keep_debug=1)
    _load(cd, slam, st, torch)
    rep = slam.step(torch.as_tensor(y64, device="cuda:0"))
    _, ref = OS.step(base, st, y64.astype(np.complex128), prm)
    assert rep["n_feat"] == ref["n_slots"] == 9
    assert rep["ident"] == [f["ident"] for f in ref["features"]]
    slam.close()
    # (b) a snapshot without power: the proposal has no residual to place a PF on (EZEROMASS), no birth
    cfg2 = small_cfg(J=1, K=1, ny=4, nv=4, nf=16, P=64, index=5)
    sc2 = scenes.make_scene(cfg2)
    base2 = orc.Oracle.from_scene(sc2)
    _, eta2 = orc.measurement(base2, sc2, scenes.P_TRUE)
    y264 = np.zeros((cfg2.J, cfg2.nf, cfg2.Na), dtype=np.complex64)
    prm2 = OS.Params(P_m=32, N_g=256)
    st2 = _known_state(OS, cfg2, sc2, P, eta2, weak=False)
    scene2 = cd.Scene.from_synthetic(sc2, precision="fp64")
    slam2 = cd.Slam(ctx, scene2, P, P_m=prm2.P_m, N_g=prm2.N_g, key=prm2.key, keep_debug=1)
    _load(cd, slam2, st2, torch)
    rep2 = slam2.step(torch.as_tensor(y264, device="cuda:0"))
    _, ref2 = OS.step(base2, st2, y264.astype(np.complex128), prm2)
    assert rep2["n_feat"] == ref2["n_slots"] == len(st2.slots)
    slam2.close()


def test_slam_rejects_bad_arguments(cd, ctx):
    cfg = small_cfg(J=1, K=1, ny=4, nv=4, nf=16, P=64, index=5)
    scene = cd.Scene.from_synthetic(scenes.make_scene(cfg))
    with pytest.raises(cd.CdmsError):
        cd.Slam(ctx, scene, 0)
    with pytest.raises(cd.CdmsError):
        cd.Slam(ctx, scene, 64, c_eta=0.5)          # Marsaglia-Tsang needs c >= 1
    slam = cd.Slam(ctx, scene, 64)
    with pytest.raises(cd.CdmsError):
        slam.set_slots([0], np.zeros((1, 1)), n=0)   # time index starts at 1
    slam.close()


def test_slam_checkpoint_resume_is_bit_exact(cd, ctx, orc):
    """Checkpoint / resume: the state is the device arrays plus the host side in cdms_slam_view; a
    fresh driver restored from a checkpoint continues bit for bit (every draw is counter-based, every reduction has a
    fixed order)."""
    import torch
    cfg = small_cfg(J=2, K=2, ny=4, nv=4, nf=16, P=64, index=5)
    sc = scenes.make_scene(cfg)
    base = orc.Oracle.from_scene(sc)
    y, eta = orc.measurement(base, sc, scenes.P_TRUE)
    dy = torch.as_tensor(y.astype(np.complex64), device="cuda:0")
    scene = cd.Scene.from_synthetic(sc)
    P = 1024
    rng = np.random.default_rng(4)
    x0 = np.zeros((P, 6))
    x0[:, :3] = scenes.P_TRUE + 0.01 * rng.standard_normal((P, 3))
    a = cd.Slam(ctx, scene, P, P_m=64, N_g=512)
    a.init(torch.as_tensor(x0, device="cuda:0"), torch.full((cfg.J, P), eta, dtype=torch.float64, device="cuda:0"))
    for _ in range(2):
        a.step(dy)
    ck = a.checkpoint()
    ra = [a.step(dy) for _ in range(2)]
    va = a.view()
    b = cd.Slam(ctx, scene, P, P_m=64, N_g=512)
    b.restore(ck)
    rb = [b.step(dy) for _ in range(2)]
    vb = b.view()
    for k in ("x", "eta", "phi", "mu", "gamma", "w"):
        assert torch.equal(va[k], vb[k]), k
    for p, q in zip(ra, rb):
        assert p["ident"] == q["ident"] and np.array_equal(p["exist"], q["exist"]) and np.array_equal(p["est"], q["est"])
    a.close()
    b.close()
