"""Small shared helpers for the tests (scene construction only; no method arithmetic)."""
import math

import numpy as np

from paper_2604_19723_b200 import scenes

C = scenes.C_LIGHT


def small_cfg(J=1, K=2, ny=4, nv=4, nf=16, P=64, fc=6.5e9, B=500e6, index=90):
    return scenes.custom_config("t", J=J, K=K, ny=ny, nv=nv, nf=nf, P=P, fc=fc, B=B, index=index)


def tiny_scene(J=1, K=2, ny=4, nv=4, nf=16, P=64, fc=6.5e9, B=500e6, index=90):
    cfg = small_cfg(J, K, ny, nv, nf, P, fc, B, index)
    return scenes.make_scene(cfg), cfg


def random_rotation(rng):
    """Haar-ish random SO(3) matrix from a QR of a Gaussian matrix."""
    A = rng.standard_normal((3, 3))
    Q, R = np.linalg.qr(A)
    Q = Q @ np.diag(np.sign(np.diag(R)))
    if np.linalg.det(Q) < 0:
        Q[:, 0] = -Q[:, 0]
    return Q


def reflect(p, s):
    """Reflection of point p across the wall of SFV s, built from the wall point w = s/2 and the
    unit normal n = s/||s|| -- independent of the oracle's Householder / VA formulas."""
    n = s / np.linalg.norm(s)
    w = s / 2.0
    return p - 2.0 * np.dot(p - w, n) * n


def wrap(x):
    return (x + math.pi) % (2 * math.pi) - math.pi
