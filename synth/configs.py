"""BASELINE.json configs C1-C5 as seeded synthetic inputs.

Input generation only.  Each config yields a mesh (synth.mesh.TetMesh), the
physical constants, and the initial-condition recipe; ``initial_state`` turns a
node-coordinate array into the conserved state by the stated recipe (Gaussian
isentropic pressure pulses at rest):

    p   = p0 (1 + sum_i A_i exp(-|x - x_i|^2 / w^2))   (minimum image if periodic)
    rho = rho0 (p / p0)^(1/gamma),   u = v = w = 0,   E = p / (gamma - 1)

Units (A5): C1 is SI as BASELINE.json states it (rho0 = 1.225, p0 = 101325);
C2-C5 use the paper's scaled units of Eq. 3: p0 = 1, rho0 = 1.4,
c0 = 1, E0 = 2.5.  Seeds (A8): numpy default_rng(config index).

``scale`` shrinks a config's hex counts for oracle-sized parity runs while
keeping its geometry, boundary tags, order and pulse recipe.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import mesh as M

GAMMA = 1.4
SCALED = dict(rho0=1.4, p0=1.0)          # Eq. 3
SI = dict(rho0=1.225, p0=101325.0)       # C1 as stated


@dataclass
class Config:
    name: str
    order: int
    mesh: M.TetMesh
    rho0: float
    p0: float
    gamma: float
    pulses: list                 # [(amp, width, (cx, cy, cz)), ...]
    steps: int
    cfl: float = 0.5
    meta: dict = field(default_factory=dict)

    @property
    def q_inf(self):
        """Ambient state (Eq. 3 in scaled units): the pass-through ghost."""
        return (self.rho0, 0.0, 0.0, 0.0, self.p0 / (self.gamma - 1.0))

    @property
    def Np(self) -> int:
        N = self.order
        return (N + 1) * (N + 2) * (N + 3) // 6

    @property
    def dofs(self) -> int:
        return self.mesh.K * self.Np * 5


def initial_state(cfg: Config, x: np.ndarray) -> np.ndarray:
    """Conserved state (5, K, Np) at node coordinates x (3, K, Np) by the A7 recipe."""
    x = np.asarray(x, dtype=np.float64)
    bump = np.zeros(x.shape[1:])
    period = cfg.mesh.period
    for amp, width, c in cfg.pulses:
        d2 = np.zeros(x.shape[1:])
        for d in range(3):
            dx = x[d] - c[d]
            if period is not None and period[d] is not None:
                L = period[d]
                dx = dx - L * np.round(dx / L)
            d2 += dx * dx
        bump += amp * np.exp(-d2 / (width * width))
    p = cfg.p0 * (1.0 + bump)
    rho = cfg.rho0 * (p / cfg.p0) ** (1.0 / cfg.gamma)
    zero = np.zeros_like(p)
    return np.stack([rho, zero, zero, zero, p / (cfg.gamma - 1.0)])


def c1(scale: float = 1.0) -> Config:
    n = max(3, int(round(4 * scale)))
    m = M.kuhn_box((n, n, n), (0, 0, 0), (1, 1, 1), periodic=(True, True, True))
    return Config("C1", 2, m, gamma=GAMMA, pulses=[(0.01, 0.1, (0.5, 0.5, 0.5))], steps=10, **SI)


def c2(scale: float = 1.0) -> Config:
    n = max(2, int(round(16 * scale)))
    m = M.kuhn_box((n, n, n), (-1, -1, -1), (1, 1, 1), bc_tag=M.BC_PASSTHROUGH)
    rng = np.random.default_rng(2)
    while True:                                   # uniform in the ball |x| < 0.3
        c = rng.uniform(-0.3, 0.3, size=3)
        if np.linalg.norm(c) < 0.3:
            break
    return Config("C2", 3, m, gamma=GAMMA, pulses=[(0.005, 0.05, tuple(c.tolist()))], steps=200, **SCALED)


def c3(scale: float = 1.0) -> Config:
    n = max(4, int(round(48 * scale)))
    # octant-mirrored Kuhn split: under the cubed-ball map the plain split puts all four
    # vertices of some cube-corner/edge tets on the sphere (h_min / h_median 4e-4)
    m = M.kuhn_box((n, n, n), (-1, -1, -1), (1, 1, 1), bc_tag=M.BC_PASSTHROUGH, mirror=True)
    m = M.carve_horn(M.cubed_ball(m, 1.0))
    return Config("C3", 3, m, gamma=GAMMA, pulses=[(0.10, 0.05, (-0.5, 0.0, 0.0))], steps=500, **SCALED)


def c4(scale: float = 1.0, nparts: int = 1) -> Config:
    nx, ny = max(4, int(round(64 * scale))), max(4, int(round(62 * scale)))
    m = M.kuhn_box((nx, ny, ny), (-0.5, -1, -1), (1.5, 1, 1), bc_tag=M.BC_PASSTHROUGH)
    m = M.carve_horn(m)
    cfg = Config("C4", 4, m, gamma=GAMMA, pulses=[(0.10, 0.05, (0.6, 0.0, 0.0))], steps=1000, **SCALED)
    cfg.meta["nparts"] = nparts
    return cfg


def c5(scale: float = 1.0, nparts: int = 1) -> Config:
    n = max(3, int(round(40 * scale)))
    m = M.kuhn_box((n * nparts, n, n), (0, 0, 0), (nparts, 1, 1), periodic=(True, True, True))
    rng = np.random.default_rng(5)
    pulses = []
    for p in range(nparts):                        # 8 pulses per unit cube (A17)
        for _ in range(8):
            amp = rng.uniform(0.001, 0.005)
            c = rng.uniform(0.0, 1.0, size=3) + np.array([p, 0.0, 0.0])
            pulses.append((float(amp), 0.1, tuple(c.tolist())))
    cfg = Config("C5", 6, m, gamma=GAMMA, pulses=pulses, steps=100, **SCALED)
    cfg.meta["nparts"] = nparts
    return cfg


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def make(name: str, scale: float = 1.0, **kw) -> Config:
    return CONFIGS[name](scale=scale, **kw)
