"""Oracle pins for row A1 (anchor geometry): P:L29-61."""
import numpy as np
import pytest

from paper_2604_19723_b200 import scenes
from tests.helpers import random_rotation, reflect, tiny_scene


def test_pa_rotations_in_so3():
    # R_j in SO(3) (P:L49-50, P:L2116 fn)
    sc = scenes.make_scene(scenes.CONFIGS["c5"])
    for R in sc.pa_rot:
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-12)
        assert abs(np.linalg.det(R) - 1.0) < 1e-12


def test_householder_invariants(orc):
    # H = H^T, H^2 = I, det H = -1, H s = -s
    sc, cfg = tiny_scene(K=8, J=4)
    o = orc.Oracle.from_scene(sc)
    st, lay, va, H = o.layout(sc.sfv)
    assert st == 0
    assert np.allclose(H[0], np.eye(3))
    for k in range(1, o.S):
        Hk = H[k]
        s = sc.sfv[k - 1]
        assert np.allclose(Hk, Hk.T, atol=1e-15)
        assert np.allclose(Hk @ Hk, np.eye(3), atol=1e-14)
        assert abs(np.linalg.det(Hk) + 1.0) < 1e-13
        assert np.allclose(Hk @ s, -s, atol=1e-13)


def test_wall_from_sfv_reflects_origin_onto_sfv():
    # wall point w = s/2, normal n = s/||s||: reflecting the origin gives s
    for s in scenes.WALL_SFV:
        assert np.allclose(reflect(np.zeros(3), s), s, atol=1e-13)


def test_va_is_reflection_of_pa(orc):
    # p_VA equals the reflection of p_j across the wall plane
    sc, cfg = tiny_scene(K=8, J=4)
    o = orc.Oracle.from_scene(sc)
    st, lay, va, H = o.layout(sc.sfv)
    for j in range(o.J):
        assert np.allclose(va[j, 0], sc.pa_pos[j])
        for k in range(1, o.S):
            assert np.allclose(va[j, k], reflect(sc.pa_pos[j], sc.sfv[k - 1]), atol=1e-12)


def test_va_special_cases(orc):
    rng = np.random.default_rng(3)
    s = np.array([1.5, -2.0, 0.7])
    # PA at the origin -> VA = s; PA on the plane -> VA = PA; VA of VA = PA
    for pj, expect in [(np.zeros(3), s), (s / 2.0, s / 2.0)]:
        o = orc.Oracle(pj[None, :], np.eye(3)[None], 2, 2, 0.01, 0.01, [6.5e9, 6.6e9], 6.55e9, K=1)
        st, lay, va, H = o.layout(s[None, :])
        assert np.allclose(va[0, 1], expect, atol=1e-14)
    pj = rng.standard_normal(3)
    o = orc.Oracle(pj[None, :], np.eye(3)[None], 2, 2, 0.01, 0.01, [6.5e9, 6.6e9], 6.55e9, K=1)
    st, lay, va, H = o.layout(s[None, :])
    o2 = orc.Oracle(va[0, 1][None, :], np.eye(3)[None], 2, 2, 0.01, 0.01, [6.5e9, 6.6e9], 6.55e9, K=1)
    st, lay2, va2, H2 = o2.layout(s[None, :])
    assert np.allclose(va2[0, 1], pj, atol=1e-13)


def test_zero_sfv_is_invalid(orc):
    # p_sfv in R^3 \ {0}
    o = orc.Oracle(np.zeros((1, 3)), np.eye(3)[None], 2, 2, 0.01, 0.01, [6.5e9, 6.6e9], 6.55e9, K=1)
    st, *_ = o.layout(np.zeros((1, 3)))
    assert st == orc.EINVAL


def test_template_and_layout_columns(orc):
    # P~ symmetric about the origin in the yz plane, column m = iy*nv + iv;
    # VA layout column m = reflection of PA layout column m
    rng = np.random.default_rng(5)
    ny, nv, dy, dv = 3, 5, 0.02, 0.03
    R = random_rotation(rng)
    pj = np.array([0.3, -1.0, 2.0])
    sfv = np.array([[4.0, 1.0, -0.5], [0.0, -3.0, 0.0]])
    o = orc.Oracle(pj[None], R[None], ny, nv, dy, dv, [6.5e9, 6.6e9], 6.55e9, K=2)
    pt = o.template()
    assert np.allclose(pt[0], 0.0)
    assert np.allclose(pt.sum(axis=1), 0.0, atol=1e-15)
    for iy in range(ny):
        for iv in range(nv):
            m = iy * nv + iv
            assert np.isclose(pt[1, m], (iy - (ny - 1) / 2) * dy)
            assert np.isclose(pt[2, m], (iv - (nv - 1) / 2) * dv)
    st, lay, va, H = o.layout(sfv)
    assert st == 0
    pa_cols = pj[:, None] + R @ pt
    assert np.allclose(lay[0, 0], pa_cols, atol=1e-14)
    for k in range(1, 3):
        for m in range(ny * nv):
            assert np.allclose(lay[0, k][:, m], reflect(pa_cols[:, m], sfv[k - 1]), atol=1e-12)


def test_local_ray_norm(orc):
    # ||r'|| = ||p - p_VA||; LOS r' = R^T (p - p_j)
    import ctypes as C
    rng = np.random.default_rng(9)
    R = random_rotation(rng)
    pj = np.array([1.0, 2.0, 0.5])
    s = np.array([0.0, 7.0, 0.0])
    o = orc.Oracle(pj[None], R[None], 2, 2, 0.01, 0.01, [6.5e9, 6.6e9], 6.55e9, K=1)
    st, lay, va, H = o.layout(s[None])
    p = np.array([0.2, 1.1, -0.3])
    dp = C.POINTER(C.c_double)
    for k in range(2):
        rl = np.zeros(3)
        Hk = np.ascontiguousarray(H[k])
        vak = np.ascontiguousarray(va[0, k])
        orc.lib().orc_local_ray(C.byref(o.sc), 0, Hk.ctypes.data_as(dp), vak.ctypes.data_as(dp),
                                p.ctypes.data_as(dp), rl.ctypes.data_as(dp))
        assert np.isclose(np.linalg.norm(rl), np.linalg.norm(p - va[0, k]), rtol=1e-14)
        if k == 0:
            assert np.allclose(rl, R.T @ (p - pj), atol=1e-14)
