"""Seeded synthetic scene inputs for the coherent-likelihood hot path.

This module draws RANDOM NUMBERS and fixes scene constants only.  It holds none of
the method's arithmetic: no array response, no likelihood, no weights.  Both the
fp64 oracle (``oracle/``, via the tests) and the CUDA path (via ``bench.py``) build
the measurement y = sum_s rho_s psi_s(p_true) + sqrt(eta) w from these draws with
their OWN response code ("Input recipe").

Scene recipe (PAPER.md P:L3668-3830 for the shapes):
  * c = 299 792 458 m/s, f_c = 6.5 GHz, B = 500 MHz, Delta_f = B/(N_f-1)
    (N_f = B/Delta_f + 1), URA spacing lambda/2.
  * walls as SFVs s_k = 2 a n (wall at distance a, unit normal n).
  * PAs with R_j = R_z(psi_j) R_y(10 deg).
  * amplitudes rho_0 = e^{j phi_0}, rho_k = 0.5 e^{j phi_k}, shared by all PAs
    (coherent premise); SNR = P_ch / eta = 100 (20 dB).
  * NZM priors m_js = rho_s (1 + 0.05 xi_js), v_js = 0.1 |rho_s|^2; ZM: m = 0,
    v = |rho_s|^2.
  * particles: 1/2 N(p_true, 0.05^2 I) + 1/2 U(ROI), velocities N(0, 0.5^2 I);
    ROI x in [-3.5, 4.5], y in [-1, 4.5], z in [-1, 1] (reading C-amb-19).

Particles are drawn in blocks of ``BLOCK`` with one PCG64 stream per block, so a
rank can draw exactly its own shard and the global set does not depend on the
number of ranks.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

C_LIGHT = 299_792_458.0
BLOCK = 65536
BASE_SEED = 2604197230

# SFVs of the walls k1..k8: wall at distance a with unit normal n -> s = 2 a n
_S2 = 1.0 / math.sqrt(2.0)
WALL_SFV = np.array([
    [-9.0, 0.0, 0.0],                 # k1: x = -4.5
    [11.0, 0.0, 0.0],                 # k2: x = 5.5
    [0.0, -4.0, 0.0],                 # k3: y = -2
    [0.0, 11.0, 0.0],                 # k4: y = 5.5
    [0.0, 0.0, -3.0],                 # k5: floor z = -1.5
    [0.0, 0.0, 5.0],                  # k6: ceiling z = 2.5
    [13.0 * _S2, 13.0 * _S2, 0.0],    # k7: n = (1,1,0)/sqrt2, a = 6.5
    [-12.0 * _S2, 12.0 * _S2, 0.0],   # k8: n = (-1,1,0)/sqrt2, a = 6.0
])

PA_POS = np.array([
    [-4.0, 1.75, 0.5],
    [5.0, 1.75, 0.5],
    [0.5, -1.5, 0.5],
    [0.5, 5.0, 0.5],
    # PA5..PA8 (J > 4, only the J = 8 edge-shape tests use them): the room's corners at 1.5 m, facing inwards,
    # on the inner side of every wall k1..k8
    [-4.0, -1.5, 1.5],
    [5.0, -1.5, 1.5],
    [4.5, 4.2, 1.5],
    [-3.8, 4.2, 1.5],
])
PA_YAW_DEG = np.array([0.0, 180.0, 90.0, -90.0, 45.0, 135.0, -135.0, -45.0])
PA_TILT_DEG = 10.0

P_TRUE = np.array([0.7, 1.9, 0.2])
V_TRUE = np.array([0.5, 0.2, 0.0])
ROI_LO = np.array([-3.5, -1.0, -1.0])
ROI_HI = np.array([4.5, 4.5, 1.0])


def rot_z(deg: float) -> np.ndarray:
    a = math.radians(deg)
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def rot_y(deg: float) -> np.ndarray:
    a = math.radians(deg)
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    index: int
    J: int
    K: int
    ny: int
    nv: int
    nf: int
    P: int
    fc: float = 6.5e9
    B: float = 500e6
    steps: int = 1
    wavefront: str = "spherical"

    @property
    def S(self) -> int:
        return self.K + 1

    @property
    def Na(self) -> int:
        return self.ny * self.nv

    @property
    def Nz(self) -> int:
        return self.nf * self.Na

    @property
    def df(self) -> float:
        return self.B / (self.nf - 1) if self.nf > 1 else 0.0

    @property
    def lam(self) -> float:
        return C_LIGHT / self.fc

    @property
    def seed(self) -> int:
        return BASE_SEED + self.index

    def f_pb(self) -> np.ndarray:
        """Passband grid f_pb = f_c 1 + f, f = [-(N_f-1)/2 .. (N_f-1)/2] Delta_f."""
        k = np.arange(self.nf, dtype=np.float64)
        return self.fc + (k - (self.nf - 1) / 2.0) * self.df

    def evals_per_step(self) -> int:
        return self.P * self.J * self.S


CONFIGS = {
    "c1": Config("c1", 0, J=1, K=2, ny=4, nv=4, nf=16, P=1000, steps=10),
    "c2": Config("c2", 1, J=1, K=4, ny=8, nv=8, nf=128, P=100_000),
    "c3": Config("c3", 2, J=2, K=6, ny=8, nv=8, nf=512, P=1_000_000),
    "c4": Config("c4", 3, J=1, K=4, ny=16, nv=16, nf=256, P=1_000_000),
    "c5": Config("c5", 4, J=4, K=8, ny=8, nv=8, nf=1024, P=16_000_000),
    # paper Experiment-1 shape (context only): f_c 3.5 GHz, B 100 MHz
    "exp1": Config("exp1", 5, J=4, K=4, ny=4, nv=4, nf=10, P=30_000, fc=3.5e9, B=100e6),
}


def custom_config(name: str = "custom", *, J: int, K: int, ny: int, nv: int, nf: int, P: int,
                  fc: float = 6.5e9, B: float = 500e6, index: int = 99) -> Config:
    return Config(name, index, J=J, K=K, ny=ny, nv=nv, nf=nf, P=P, fc=fc, B=B)


@dataclasses.dataclass
class Scene:
    """Everything the hot path consumes except the measurement y itself."""
    cfg: Config
    pa_pos: np.ndarray      # [J][3]
    pa_rot: np.ndarray      # [J][3][3]
    sfv: np.ndarray         # [K][3]
    dy: float
    dv: float
    rho: np.ndarray         # [S] complex: true amplitudes, shared across PAs
    xi: np.ndarray          # [J][S] complex CN(0,1): prior perturbation draws
    noise_unit: np.ndarray  # [J][nf][Na] complex CN(0,1) (paper vec order: k slow, m fast)
    u_bits: int             # 32-bit uniform for systematic resampling
    philox_key: int         # 64-bit key for bp_step's counter-based RNG


def make_scene(cfg: Config, step: int = 0) -> Scene:
    """Draw order (PCG64, seed = seed_c): amplitude phases, prior perturbations,
    [particles are drawn separately by make_particles], noise per PA, u_bits."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([cfg.seed, 0, step])))
    J, S = cfg.J, cfg.S
    phases = rng.uniform(0.0, 2.0 * math.pi, size=S)
    rho = np.exp(1j * phases) * np.where(np.arange(S) == 0, 1.0, 0.5)
    xi = (rng.standard_normal((J, S)) + 1j * rng.standard_normal((J, S))) / math.sqrt(2.0)
    noise = np.empty((J, cfg.nf, cfg.Na), dtype=np.complex128)
    for j in range(J):
        re = rng.standard_normal((cfg.nf, cfg.Na))
        im = rng.standard_normal((cfg.nf, cfg.Na))
        noise[j] = (re + 1j * im) / math.sqrt(2.0)   # CN(0,1): re, im iid N(0, 1/2) (C-amb-20)
    u_bits = int(rng.integers(0, 2**32, dtype=np.uint64))
    pa_rot = np.stack([rot_z(PA_YAW_DEG[j]) @ rot_y(PA_TILT_DEG) for j in range(J)])
    return Scene(cfg=cfg, pa_pos=PA_POS[:J].copy(), pa_rot=pa_rot, sfv=WALL_SFV[:cfg.K].copy(),
                 dy=cfg.lam / 2.0, dv=cfg.lam / 2.0, rho=rho, xi=xi, noise_unit=noise,
                 u_bits=u_bits, philox_key=cfg.seed)


def priors(scene: Scene, mode: str = "nzm") -> tuple[np.ndarray, np.ndarray]:
    """Per-(j,s) amplitude prior (m, v): NZM m = rho(1+0.05 xi), v = 0.1|rho|^2; ZM m = 0, v = |rho|^2."""
    rho = scene.rho[None, :]
    if mode == "nzm":
        m = rho * (1.0 + 0.05 * scene.xi)
        v = np.broadcast_to(0.1 * np.abs(rho) ** 2, m.shape).copy()
    elif mode == "zm":
        m = np.zeros_like(scene.xi)
        v = np.broadcast_to(np.abs(rho) ** 2, m.shape).copy()
    else:
        raise ValueError(mode)
    return m, v


def _particle_block(cfg: Config, block: int, n: int, spread: float = 0.05) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([cfg.seed, 1, block])))
    pick = rng.uniform(size=n) < 0.5
    near = P_TRUE[None, :] + spread * rng.standard_normal((n, 3))
    far = ROI_LO[None, :] + (ROI_HI - ROI_LO)[None, :] * rng.uniform(size=(n, 3))
    x = np.empty((n, 6))
    x[:, :3] = np.where(pick[:, None], near, far)
    x[:, 3:] = 0.5 * rng.standard_normal((n, 3))
    return x


def make_particles(cfg: Config, start: int = 0, count: Optional[int] = None) -> np.ndarray:
    """Particles [start, start+count) of the config's global set, float64 [count][6]
    (x, y, z, vx, vy, vz).  Identical rows whatever the shard boundaries.  Requests reaching past cfg.P (a larger
    particle set than the config's) draw whole blocks of BLOCK rows throughout."""
    if count is None:
        count = cfg.P - start
    out = np.empty((count, 6))
    end = cfg.P if start + count <= cfg.P else start + count + BLOCK
    b0, b1 = start // BLOCK, (start + count - 1) // BLOCK if count > 0 else start // BLOCK - 1
    for b in range(b0, b1 + 1):
        lo, hi = b * BLOCK, min((b + 1) * BLOCK, end)
        blk = _particle_block(cfg, b, hi - lo)
        s, e = max(lo, start), min(hi, start + count)
        out[s - start:e - start] = blk[s - lo:e - lo]
    return out


def stratified_sample(P: int, n: int, seed: int = 7) -> np.ndarray:
    """Indices for parity checks on big configs: every floor(P/n)-th particle."""
    if n >= P:
        return np.arange(P)
    step = P // n
    return np.arange(0, step * n, step)
