"""F3: cdms_birth_proposal (birth.cu + the likelihood engine) against the fp64 oracle's
orc_birth_proposal on identical seeded inputs.

Tolerances: candidates bit-exact (same Philox words and the same uncontracted fp64 arithmetic);
P_B within 1e-5 (FP32) / 1e-8 (FP64) of max P_B -- the correlations carry the likelihood engine's
c error (~1e-7 relative, section 8) doubled by |.|^2, and in FP64 mode the residual z~ is handed to the
engine as a complex64 snapshot (the ABI's snapshot type), one rounding of 2^-24 per element; i* equal whenever
the oracle's two largest P_B differ by more than twice that bound (otherwise either is a valid mode and the
GPU's must be within the bound of the max); mu = p_{i*} exactly; C within 1e-4 (FP32) / 1e-7 (FP64) of ||C||
when the modes agree."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import oracle as orc_mod
from paper_2604_19723_b200 import scenes
from tests.gpu_common import record
from tests.helpers import small_cfg
from tests.test_parity_gpu import cd, ctx  # noqa: F401  (fixtures)

TOL_PB = {"fp32": 1e-5, "fp64": 1e-8}
TOL_C = {"fp32": 1e-4, "fp64": 1e-7}


class BirthCase:
    def __init__(self, orc, cfg, wavefront="spherical", precision="fp32", L=2, N_g=400, key=77, counter=5,
                 pathloss=False, box_half=0.4, x_offset=(0.01, -0.02, 0.005)):
        import torch
        from paper_2604_19723_b200 import cdms
        self.cfg = cfg
        self.sc = scenes.make_scene(cfg)
        self.o = orc.Oracle.from_scene(self.sc, wavefront=wavefront, pathloss=pathloss)
        y, _ = orc.measurement(self.o, self.sc, scenes.P_TRUE, wavefront=None)
        self.y64 = y.astype(np.complex64)
        self.y = self.y64.astype(np.complex128)
        self.x_hat = scenes.P_TRUE + np.array(x_offset)
        self.sl = self.sc.sfv[:L]
        target = self.sc.sfv[min(L, cfg.K - 1)]
        self.box = np.concatenate([target - box_half, target + box_half])
        self.N_g, self.key, self.counter = N_g, key, counter
        self.scene = cdms.Scene.from_synthetic(self.sc, wavefront=wavefront, pathloss=pathloss, precision=precision)
        self.dy = torch.as_tensor(self.y64, device="cuda:0").contiguous()

    def gpu(self, ctx):
        from paper_2604_19723_b200 import cdms
        out, pb, cand = cdms.birth_proposal(ctx, self.scene, self.x_hat, self.sl, self.dy, self.box, self.N_g,
                                            self.key, self.counter)
        ctx.sync()
        return out.cpu().numpy(), pb.cpu().numpy(), cand.cpu().numpy()

    def oracle(self):
        return self.o.birth_proposal(self.x_hat, self.sl, self.y.reshape(self.cfg.J, -1), self.box, self.N_g,
                                     self.key, self.counter)


def check_birth(case, ctx, precision):
    out, pb, cand = case.gpu(ctx)
    st, pbo, cando, muo, Co, isto = case.oracle()
    assert st == 0
    assert np.array_equal(cand, cando), "candidates must be bit-exact"
    scale = pbo.max()
    e_pb = np.max(np.abs(pb - pbo)) / scale
    record("birth_pb_rel", e_pb, TOL_PB[precision], precision=precision, config=case.cfg.name)
    assert e_pb <= TOL_PB[precision], e_pb
    ist = int(out[12])
    top2 = np.sort(pbo)[-2:] if len(pbo) > 1 else np.array([0.0, scale])
    if (top2[1] - top2[0]) > 2 * TOL_PB[precision] * scale:
        assert ist == isto, (ist, isto)
    else:
        assert pbo[ist] >= scale * (1 - 2 * TOL_PB[precision])
    assert np.array_equal(out[:3], cand[ist])
    if ist == isto:
        e_c = np.max(np.abs(out[3:12].reshape(3, 3) - Co)) / max(np.linalg.norm(Co), 1e-300)
        record("birth_C_rel", e_c, TOL_C[precision], precision=precision, config=case.cfg.name)
        assert e_c <= TOL_C[precision], e_c
    return out, pb, cand


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("wf", ["spherical", "planar_wb", "planar_nb"])
def test_birth_parity(cd, ctx, orc, wf, precision):
    cfg = small_cfg(J=2, K=4, ny=4, nv=4, nf=64, P=1, index=97)
    check_birth(BirthCase(orc, cfg, wavefront=wf, precision=precision), ctx, precision)


@pytest.mark.parametrize("shape,L", [
    (dict(J=3, K=3, ny=3, nv=5, nf=100, P=1), 0),     # LOS-only projector, ragged antennas / subcarriers
    (dict(J=1, K=8, ny=8, nv=8, nf=128, P=1), 7),     # L = 7 legacy PFs (Psi with 8 columns)
    (dict(J=4, K=2, ny=2, nv=2, nf=16, P=1), 1),      # J = 4
])
def test_birth_shapes(cd, ctx, orc, shape, L):
    cfg = small_cfg(**shape, index=97)
    check_birth(BirthCase(orc, cfg, L=L, N_g=2500), ctx, "fp32")  # 2 reduction blocks, ragged


def test_birth_pathloss(cd, ctx, orc):
    cfg = small_cfg(J=2, K=3, ny=4, nv=4, nf=32, P=1, index=97)
    check_birth(BirthCase(orc, cfg, pathloss=True), ctx, "fp32")


def test_birth_zero_mass_and_determinism(cd, ctx, orc):
    import torch
    cfg = small_cfg(J=1, K=2, ny=4, nv=4, nf=32, P=1, index=97)
    case = BirthCase(orc, cfg, N_g=300)
    a = case.gpu(ctx)
    b = case.gpu(ctx)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    case.dy = torch.zeros_like(case.dy)
    from paper_2604_19723_b200 import cdms
    cdms.birth_proposal(ctx, case.scene, case.x_hat, case.sl, case.dy, case.box, case.N_g, 1, 0)
    with pytest.raises(cd.CdmsError) as ei:
        ctx.sync()
    assert ei.value.status == cd.EZEROMASS


def test_birth_c2_scale_sampled(cd, ctx, orc):
    """c2 scene (J=1, K=4, 8x8 URA, 128 subcarriers) with 2^20 candidates; the oracle's definition evaluated on a
    stratified sample of candidates (residual from orc_birth_residual, responses from orc_response)."""
    cfg = scenes.CONFIGS["c2"]
    N_g = 1 << 20
    case = BirthCase(orc, cfg, L=2, N_g=N_g)
    out, pb, cand = case.gpu(ctx)
    st, zr = case.o.birth_residual(case.x_hat, case.sl, case.y.reshape(cfg.J, -1))
    assert st == 0
    idx = np.unique(np.concatenate([scenes.stratified_sample(N_g, 48), [int(out[12])]]))
    ref = np.zeros(len(idx))
    for n, i in enumerate(idx):
        p = orc_mod.birth_candidate(case.key, case.counter, int(i), case.box)
        assert np.array_equal(p, cand[i])
        acc = 0j
        for j in range(cfg.J):
            stj, psi = case.o.response(case.x_hat, j, 1, p[None])
            acc += np.vdot(zr[j], psi) / cfg.Nz
        ref[n] = abs(acc) ** 2
    e = np.max(np.abs(pb[idx] - ref)) / ref.max()
    record("birth_pb_rel", e, TOL_PB["fp32"], config="c2")
    assert e <= TOL_PB["fp32"], e
    assert pb[int(out[12])] == pb.max()
    w = pb / pb.sum()
    d = cand - out[:3]
    C = (w[:, None, None] * d[:, :, None] * d[:, None, :]).sum(0)
    assert np.allclose(out[3:12].reshape(3, 3), C, rtol=1e-9, atol=1e-15)
