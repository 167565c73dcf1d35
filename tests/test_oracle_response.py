"""Oracle pins for the array responses R1-R5."""
import json
import math
import os

import numpy as np
import pytest

from tests.helpers import C, random_rotation, reflect, tiny_scene, wrap

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _scene_oracle(orc, ny=4, nv=4, nf=16, fc=6.5e9, B=500e6, K=2, R=None, pj=None, pathloss=False,
                  wavefront="spherical"):
    lam = C / fc
    f_pb = fc + (np.arange(nf) - (nf - 1) / 2) * (B / (nf - 1) if nf > 1 else 0.0)
    R = np.eye(3) if R is None else R
    pj = np.zeros(3) if pj is None else pj
    return orc.Oracle(pj[None], R[None], ny, nv, lam / 2, lam / 2, f_pb, fc, K=K,
                      wavefront=wavefront, pathloss=pathloss), f_pb


@pytest.mark.parametrize("wf", ["spherical", "planar_wb", "planar_nb"])
def test_unit_modulus(orc, wf):
    # psi on the N_z-torus
    sc, cfg = tiny_scene(K=3)
    o = orc.Oracle.from_scene(sc, wavefront=wf)
    rng = np.random.default_rng(1)
    for _ in range(5):
        p = scenes_point(rng)
        for s in range(o.S):
            st, psi = o.response(p, 0, s, sc.sfv)
            assert st == 0
            assert np.allclose(np.abs(psi), 1.0, atol=1e-14)


def scenes_point(rng):
    from paper_2604_19723_b200 import scenes
    return scenes.ROI_LO + (scenes.ROI_HI - scenes.ROI_LO) * rng.uniform(size=3)


def test_spherical_equals_independent_va_geometry(orc):
    # R1 with the VA layout: distances from the MT to the mirrored antennas
    # computed by reflecting each PA antenna across the wall plane (w = s/2, n = s/||s||)
    rng = np.random.default_rng(2)
    R = random_rotation(rng)
    pj = np.array([-4.0, 1.75, 0.5])
    o, f_pb = _scene_oracle(orc, ny=3, nv=4, nf=7, K=2, R=R, pj=pj)
    sfv = np.array([[-9.0, 0.0, 0.0], [0.0, 11.0, 0.0]])
    pt = o.template()
    pa_cols = pj[:, None] + R @ pt
    p = np.array([0.7, 1.9, 0.2])
    for s in range(3):
        cols = pa_cols if s == 0 else np.stack([reflect(pa_cols[:, m], sfv[s - 1]) for m in range(12)], 1)
        d = np.linalg.norm(p[:, None] - cols, axis=0)
        expect = np.exp(-2j * np.pi * np.outer(f_pb, d) / C).reshape(-1)  # n = k*Na + m
        st, psi = o.response(p, 0, s, sfv)
        assert st == 0
        assert np.max(np.abs(wrap(np.angle(psi * np.conj(expect))))) < 1e-9


def test_planar_nb_kronecker_equals_per_element(orc):
    # R3: (b (x) a_y (x) a_z) e^{-j2 pi f_c tau} equals the per-element phase
    # -2 pi f_pb,k ||r'||/c + 2 pi p~_m^T u' / lambda
    rng = np.random.default_rng(4)
    R = random_rotation(rng)
    pj = np.array([0.5, -1.5, 0.5])
    fc = 6.5e9
    o, f_pb = _scene_oracle(orc, ny=4, nv=3, nf=9, K=1, R=R, pj=pj, wavefront="planar_nb")
    sfv = np.array([[0.0, 0.0, -3.0]])
    pt = o.template()
    st, lay, va, H = o.layout(sfv)
    lam = C / fc
    for trial in range(4):
        p = scenes_point(rng)
        for s in range(2):
            rl = R.T @ H[s] @ (p - va[0, s])
            rn = np.linalg.norm(rl)
            u = rl / rn
            ph = (-2 * np.pi * np.outer(f_pb, np.full(12, rn)) / C
                  + 2 * np.pi * (pt.T @ u)[None, :] / lam)
            st, psi = o.response(p, 0, s, sfv)
            assert st == 0
            assert np.max(np.abs(wrap(np.angle(psi) - ph.reshape(-1)))) < 1e-9


def test_far_field_one_over_d_law(orc):
    # R1 -> R2: the max phase gap is the Fresnel term ~ pi f rho_perp^2 / (c d), halving per
    # distance doubling; 4x4 at 1000 x aperture < 1e-2 rad.
    o, f_pb = _scene_oracle(orc, ny=4, nv=4, nf=16, K=0)
    aperture = 3 * (C / 6.5e9) / 2 * math.sqrt(2)
    direction = np.array([0.8, 0.36, 0.48])
    gaps = []
    for mult in [125, 250, 500, 1000]:
        p = direction / np.linalg.norm(direction) * mult * aperture
        st1, sph = o.response(p, 0, 0, np.zeros((0, 3)), "spherical")
        st2, pla = o.response(p, 0, 0, np.zeros((0, 3)), "planar_wb")
        gaps.append(np.max(np.abs(wrap(np.angle(sph * np.conj(pla))))))
    ratios = [gaps[i] / gaps[i + 1] for i in range(3)]
    assert all(1.95 < r < 2.05 for r in ratios), ratios
    assert gaps[-1] < 1e-2


def test_single_element_spherical_equals_planar(orc):
    # no aperture -> R1 == R2
    o, f_pb = _scene_oracle(orc, ny=1, nv=1, nf=8, K=1)
    sfv = np.array([[0.0, 11.0, 0.0]])
    rng = np.random.default_rng(7)
    for _ in range(4):
        p = scenes_point(rng)
        for s in range(2):
            _, a = o.response(p, 0, s, sfv, "spherical")
            _, b = o.response(p, 0, s, sfv, "planar_wb")
            assert np.max(np.abs(wrap(np.angle(a * np.conj(b))))) < 1e-10


def test_delay_and_carrier_special_cases(orc):
    # N_f = 3, tau = 1/(2 Delta_f) -> b = [-1, 1, -1]; broadside u' = (1,0,0) -> a = 1;
    # ||r'|| = integer * lambda -> carrier 1
    fc, B = 6.5e9, 200e6
    o, f_pb = _scene_oracle(orc, ny=2, nv=3, nf=3, fc=fc, B=B, K=0, wavefront="planar_nb")
    df = B / 2
    p = np.array([C / (2 * df), 0.0, 0.0])
    st, psi = o.response(p, 0, 0, np.zeros((0, 3)))
    psi = psi.reshape(3, 6)
    ratio = psi / psi[1][None, :]
    assert np.allclose(ratio, np.array([-1, 1, -1])[:, None], atol=1e-9)
    assert np.allclose(psi / psi[:, :1], 1.0, atol=1e-12)  # a = 1 at broadside
    lam = C / fc
    p = np.array([30 * lam, 0.0, 0.0])
    st, psi = o.response(p, 0, 0, np.zeros((0, 3)))
    assert np.allclose(psi.reshape(3, 6)[1], 1.0, atol=1e-9)


def test_pathloss_value(orc):
    g = json.load(open(os.path.join(GOLDEN, "pathloss.json")))
    o, f_pb = _scene_oracle(orc, ny=2, nv=2, nf=3, fc=g["fc"], B=50e6, K=0, pathloss=True,
                            wavefront="planar_nb")
    st, psi = o.response(np.array([g["range_m"], 0.0, 0.0]), 0, 0, np.zeros((0, 3)))
    assert np.allclose(np.abs(psi), g["gain"], rtol=g["rel_tol"])


def test_degenerate_ray(orc):
    # MT on the phase centre is excluded (r' != 0)
    o, f_pb = _scene_oracle(orc, ny=2, nv=2, nf=3, K=0)
    st, _ = o.response(np.zeros(3), 0, 0, np.zeros((0, 3)))
    assert st == orc.EDEGENERATE
