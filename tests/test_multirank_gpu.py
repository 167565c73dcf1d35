"""GPU tests of rows A6-A9 as cdms_bp_step runs them, and of the multi-rank device path.

* cdms_bp_update runs the step's own O(P) kernels (step.cu) on log-weights given by the test, so its ancestors can be
  compared bit for bit with the oracle's orc_step_update (reading C-amb-23: masses e^{l - M}) at full sizes
  (P = 1e5, 1e6: hundreds to thousands of 512-particle blocks, the two- and three-level ancestor search).
* The multi-rank path (all-gathered block partials, device-side resampling plan, ancestor gather written straight into
  the owner rank's buffers, barrier, regularization) runs on ONE GPU through the test collective backend
  (cdms_loopback_*): R contexts, one host thread each.  With block-aligned shards it must reproduce the single-rank
  run bit for bit (l, w-derived lse / est, ancestors, particles), and it must match the oracle.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2604_19723_b200 import scenes
from tests.gpu_common import Case, record
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


def _loglik_like(rng, P, spread=60.0):
    """Log-weights shaped like the likelihood's: a large common offset, a few nats of spread, some -inf."""
    l = -1.2e6 + spread * rng.standard_normal(P) - rng.exponential(200.0, P)
    l[rng.uniform(size=P) < 0.01] = -np.inf
    return l


# ---------------------------------------------------------------------------- bp_step's kernels vs the oracle
@pytest.mark.parametrize("P", [1000, 100_000, 1_000_000])
@pytest.mark.parametrize("regularize", [False, True])
def test_bp_update_matches_oracle(cd, ctx, orc, P, regularize):
    import torch
    rng = np.random.default_rng(P + int(regularize))
    l = _loglik_like(rng, P)
    x = rng.normal(size=(P, 6))
    key, step = 0x5EED_1234_ABCD, 7
    dl = torch.as_tensor(l, device="cuda:0")
    dx = torch.as_tensor(x, device="cuda:0").contiguous()
    est, lse, anc = cd.bp_update(ctx, dl, dx, key, step, regularize=regularize, want_ancestors=True)
    ctx.sync()
    st, xo, esto, lseo, anco = orc.step_update(l, x, key, step, regularize=regularize)
    assert st == 0
    a = anc.cpu().numpy()
    record("bp_update_ancestor_mismatches", int(np.sum(a != anco)), 0, P=P)
    assert np.array_equal(a, anco)                                    # bit-exact (integer CDF, same masses)
    assert abs(lse.item() - lseo) <= 1e-13 * abs(lseo)
    assert np.allclose(est.cpu().numpy(), esto, rtol=1e-10, atol=1e-12)
    xg = dx.cpu().numpy()
    if regularize:
        # the kernel's covariance is a different-order fp64 sum of P terms (agrees to ~1e-13 relative), which the
        # regularization increment h chol(Sigma) n (|h n| up to ~1) carries
        record("bp_update_particles_abs", np.max(np.abs(xg - xo)), 1e-11, P=P)
        assert np.max(np.abs(xg - xo)) <= 1e-11
    else:
        assert np.array_equal(xg, x[anco])                             # the gathered states themselves


def test_bp_update_onehot_and_zero_mass(cd, ctx, orc):
    import torch
    P = 4099
    l = np.full(P, -np.inf)
    l[1234] = -5.0
    x = np.arange(P * 6, dtype=np.float64).reshape(P, 6)
    dx = torch.as_tensor(x, device="cuda:0").contiguous()
    est, lse, anc = cd.bp_update(ctx, torch.as_tensor(l, device="cuda:0"), dx, 3, 1, regularize=False,
                                 want_ancestors=True)
    ctx.sync()
    assert np.all(anc.cpu().numpy() == 1234) and np.all(dx.cpu().numpy() == x[1234])
    dx = torch.as_tensor(x, device="cuda:0").contiguous()
    cd.bp_update(ctx, torch.full((P,), -np.inf, dtype=torch.float64, device="cuda:0"), dx, 3, 1)
    with pytest.raises(cd.CdmsError) as ei:
        ctx.sync()
    assert ei.value.status == cd.EZEROMASS


def test_bp_step_equals_predict_loglik_update(cd, ctx, orc):
    """cdms_bp_step = predict -> loglik -> cdms_bp_update with the same kernels: with T = 0, sigma_v = 0 the prediction
    is the identity, so bp_step must equal loglik followed by bp_update bit for bit."""
    import torch
    cfg = small_cfg(J=2, K=3, ny=4, nv=4, nf=32, P=2048)
    case = Case(orc, cfg, precision="fp64")
    key = case.sc.philox_key
    xa = case.dx.clone()
    est_a, lse_a = cd.bp_step(ctx, case.scene, xa, case.dsfv, case.dy, case.m, case.v, case.eta, 0.0, 0.0, key, 2)
    xp = case.dx.clone()
    l = cd.loglik(ctx, case.scene, xp, case.dsfv, case.dy, case.m, case.v, case.eta)
    est_b, lse_b, _ = cd.bp_update(ctx, l, xp, key, 2)
    ctx.sync()
    assert torch.equal(xa, xp) and torch.equal(est_a, est_b) and torch.equal(lse_a, lse_b)


# ---------------------------------------------------------------------------- multi-rank device path, one GPU
def _run_ranks(R, fn):
    """Run fn(rank) on R threads (each drives its own context's collective calls); re-raise the first error."""
    import torch
    torch.cuda.synchronize()  # inputs made on the default stream are ready for the ranks' own streams
    out, errs = [None] * R, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(R)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


def _group(cd, R):
    import torch
    grp = cd.LoopbackGroup(R)
    ctxs = []
    for r in range(R):
        c = cd.Context(0, torch.cuda.Stream(device=0))
        c.comm_init_loopback(grp, r)
        ctxs.append(c)
    return grp, ctxs


@pytest.mark.parametrize("R", [2, 4])
def test_loopback_bp_step_bit_identical_to_one_rank(cd, orc, R):
    """Block-aligned shards (P_local = 3 x 512): R ranks reproduce the 1-rank bp_step on all P_total particles bit
    for bit over three steps -- lse, est, every particle (ancestors + regularization) -- and l of the first step."""
    import torch
    P_local = 1536
    cfg = small_cfg(J=2, K=3, ny=4, nv=4, nf=64, P=P_local * R)
    case = Case(orc, cfg)
    key = case.sc.philox_key
    one = cd.Context(0)
    x1 = case.dx.clone()
    ref = []
    for n in range(3):
        e, s = cd.bp_step(one, case.scene, x1, case.dsfv, case.dy, case.m, case.v, case.eta, 0.1, 0.5, key, n)
        one.sync()
        ref.append((e.clone(), s.clone(), x1.clone()))
    one.close()
    grp, ctxs = _group(cd, R)
    shards = [case.dx[r * P_local:(r + 1) * P_local].clone() for r in range(R)]

    def rank_fn(r):
        c = ctxs[r]
        with torch.cuda.stream(c.stream):
            res = []
            for n in range(3):
                e, s = cd.bp_step(c, case.scene, shards[r], case.dsfv, case.dy, case.m, case.v, case.eta, 0.1, 0.5,
                                  key, n)
                c.sync()
                res.append((e.clone(), s.clone(), shards[r].clone()))
            return res

    got = _run_ranks(R, rank_fn)
    for n in range(3):
        e1, s1, x_ref = ref[n]
        for r in range(R):
            e, s, xr = got[r][n]
            assert torch.equal(e, e1) and torch.equal(s, s1), (n, r)
        xall = torch.cat([got[r][n][2] for r in range(R)])
        assert torch.equal(xall, x_ref), n
    for c in ctxs:
        c.close()
    grp.close()


@pytest.mark.parametrize("R,P_local", [(2, 1000), (4, 2048), (3, 777)])
def test_loopback_bp_update_matches_oracle(cd, orc, R, P_local):
    """Any shard size: every rank's ancestors (global ids of its slots) and states equal the oracle's single-process
    orc_step_update on the concatenated l (ancestors bit-exact; regularized particles within 1e-12)."""
    import torch
    P = R * P_local
    rng = np.random.default_rng(R * 1000 + P_local)
    l = _loglik_like(rng, P, spread=8.0)
    x = rng.normal(size=(P, 6))
    key, step = 99, 5
    st, xo, esto, lseo, anco = orc.step_update(l, x, key, step)
    assert st == 0
    grp, ctxs = _group(cd, R)

    def rank_fn(r):
        c = ctxs[r]
        with torch.cuda.stream(c.stream):
            dl = torch.as_tensor(l[r * P_local:(r + 1) * P_local], device="cuda:0")
            dx = torch.as_tensor(x[r * P_local:(r + 1) * P_local], device="cuda:0").contiguous()
            est, lse, anc = cd.bp_update(c, dl, dx, key, step, want_ancestors=True)
            c.sync()
            return est.cpu().numpy(), lse.item(), anc.cpu().numpy(), dx.cpu().numpy()

    got = _run_ranks(R, rank_fn)
    anc = np.concatenate([g[2] for g in got])
    xg = np.concatenate([g[3] for g in got])
    assert np.array_equal(anc, anco)
    assert np.max(np.abs(xg - xo)) <= 1e-11
    for est, lse, _, _ in got:
        assert abs(lse - lseo) <= 1e-13 * abs(lseo)
        assert np.allclose(est, esto, rtol=1e-10, atol=1e-12)
    for c in ctxs:
        c.close()
    grp.close()


@pytest.mark.parametrize("R", [2, 4])
def test_loopback_resample_normalize_moments(cd, orc, R):
    """cdms_resample (global ancestors, bit-exact), cdms_weights_normalize (1e-14) and cdms_moments over R ranks."""
    import torch
    P_local = 3001
    P = R * P_local
    rng = np.random.default_rng(R)
    w = rng.exponential(size=P) * (rng.uniform(size=P) < 0.8)
    w[0] = 1.0
    l = np.log(w / w.sum())
    x = rng.normal(size=(P, 6))
    u = int(rng.integers(0, 2**32))
    st, anc_ref = orc.resample(w, u)
    st, w_ref, lse_ref = orc.normalize(l)
    st, est_ref = orc.moments(x, w_ref)
    grp, ctxs = _group(cd, R)

    def rank_fn(r):
        c = ctxs[r]
        sl = slice(r * P_local, (r + 1) * P_local)
        with torch.cuda.stream(c.stream):
            anc = cd.resample(c, torch.as_tensor(w[sl], device="cuda:0"), u)
            wn, lse = cd.weights_normalize(c, torch.as_tensor(l[sl], device="cuda:0"))
            est = cd.moments(c, torch.as_tensor(x[sl], device="cuda:0").contiguous(), wn)
            c.sync()
            return anc.cpu().numpy(), wn.cpu().numpy(), lse.item(), est.cpu().numpy()

    got = _run_ranks(R, rank_fn)
    assert np.array_equal(np.concatenate([g[0] for g in got]), anc_ref)
    wg = np.concatenate([g[1] for g in got])
    assert np.max(np.abs(wg - w_ref)) <= 1e-14 * w_ref.max()
    for _, _, lse, est in got:
        assert abs(lse - lse_ref) <= 1e-13 * max(1.0, abs(lse_ref))
        assert np.allclose(est, est_ref, rtol=1e-10, atol=1e-12)
    for c in ctxs:
        c.close()
    grp.close()
