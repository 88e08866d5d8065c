"""Workload presets (BASELINE.json configs) shared by tests, bench.py and smoke().

Pure configuration: sizes, parameters, seeds and the cube side that gives the stated
volume fraction.  It holds none of the method's arithmetic (no force, no grid, no
RNG); each side (oracle/ and the CUDA library) generates the population itself from
the per-id Philox recipe of DESIGN.md section 5.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, asdict


def side_for_fraction(n: int, mean_d3: float, phi: float) -> float:
    """Cube side such that n spheres with E[d^3] = mean_d3 fill a volume fraction phi."""
    return (n * (math.pi / 6.0) * mean_d3 / phi) ** (1.0 / 3.0)


@dataclass(frozen=True)
class MechConfig:
    name: str
    n: int
    side: float
    d_lo: float
    d_width: float          # d = d_lo + d_width*u (d_random) else d = d_lo
    d_random: bool
    steps: int
    detect_static: bool
    seed: int = 1
    dt: float = 0.01
    max_disp: float = 3.0
    k: float = 2.0
    gamma: float = 1.0
    force_threshold: float = 0.0

    def to_dict(self):
        return asdict(self)


# configs[0]: 4,096 spheres, d = 10 um, 160 um cube, R = max d, dt = 0.01, cap 3 um,
# 10 steps, seed 1, mechanics only (static skip off; R25).
CFG1 = MechConfig("cfg1", 4096, 160.0, 10.0, 0.0, False, 10, False)

# configs[1]: 10M spheres, d ~ U[8,12] um (E[d^3] = 1040 um^3), cube for 50 % volume
# fraction (side 2216.6 um), static-agent skip on, 100 steps on 1 GPU.
CFG2_MEAN_D3 = (12.0**4 - 8.0**4) / (4.0 * 4.0)
CFG2 = MechConfig("cfg2", 10_000_000, side_for_fraction(10_000_000, CFG2_MEAN_D3, 0.5),
                  8.0, 4.0, True, 100, True)


def cfg2_scaled(n: int) -> MechConfig:
    """cfg2's density and diameter mix at a smaller agent count (parity-test size)."""
    return MechConfig(f"cfg2@{n}", n, side_for_fraction(n, CFG2_MEAN_D3, 0.5), 8.0, 4.0, True,
                      100, True)


# configs[4]: 1.7B spheres, d = 10 um, 50 % volume fraction (side 12,119.7 um),
# x-slab decomposition over 1/2/4/8 GPUs, 10 steps.
CFG5 = MechConfig("cfg5", 1_700_000_000, side_for_fraction(1_700_000_000, 1000.0, 0.5),
                  10.0, 0.0, False, 10, False)

# configs[2]: cell proliferation, 1M spheres d = 8 um in a 1 mm cube, +400 um^3 per
# step, divide at d = 12 um (V >= (M_PI/6)*1728), mechanics each step, 20 steps.
CFG3 = MechConfig("cfg3", 1_000_000, 1000.0, 8.0, 0.0, False, 20, False)
CFG3_GROWTH = 400.0
CFG3_V_MAX = (math.pi / 6.0) * 1728.0


@dataclass(frozen=True)
class SirConfig:
    name: str
    n: int
    side: float           # periodic cube edge [m]
    radius: float         # infection radius [m]
    p_inf: float
    p_rec: float
    n_infected: int       # ids < n_infected start infected (R21)
    steps: int
    seed: int = 1

    def to_dict(self):
        return asdict(self)


# configs[3]: 100M point agents in a periodic 10 km cube, radius 2 m, p_inf 0.1,
# p_rec 0.01, 0.1 % initially infected, 200 steps.
CFG4 = SirConfig("cfg4", 100_000_000, 10_000.0, 2.0, 0.1, 0.01, 100_000, 200)


def cfg4_scaled(n: int, side: float = None) -> SirConfig:
    """cfg4's parameters at n agents (default: cfg4's density)."""
    if side is None:
        side = CFG4.side * (n / CFG4.n) ** (1.0 / 3.0)
    return SirConfig(f"cfg4@{n}", n, side, 2.0, 0.1, 0.01, max(1, n // 1000), 200)


@dataclass(frozen=True)
class SomaConfig:
    """SURVEY 8(f) row f4 (not one of BASELINE.json's configs): soma clustering
    (Algs. secretion_module / chemotaxis_module) with Eq. 4.3 diffusion.
    The paper's benchmark has 32k agents; its grid resolution, nu, mu and
    dt are not given, so the grid is chosen to make the stencil the measured kernel."""
    name: str
    n: int            # agents, type = id % 2
    side: float       # agents and grid cover [0, side)^3 um
    res: int          # grid points per axis (per substance)
    nu: float         # diffusion coefficient, um^2/s
    mu: float         # decay constant, 1/s
    dt: float         # s; 2 (cx+cy+cz) = 6 nu dt / dx^2 <= 1 - mu dt (explicit stability)
    q: float          # secretion_quantity
    weight: float     # gradient_weight
    d: float          # diameter (mechanics is not part of this step)
    seed: int = 1

    def to_dict(self):
        return asdict(self)


SOMA = SomaConfig("soma", 32_768, 1000.0, 512, 1.0, 0.01, 0.5, 1.0, 0.75, 10.0)

@dataclass(frozen=True)
class OncoConfig:
    """SURVEY 8(f) row f2 (not one of BASELINE.json's configs): tumor-spheroid cells
    (Alg. 4, Table 4.2 per 1 h step) at GPU scale.  Mechanics: adherence 1.8 as the force
    threshold, maximum speed 1.0 um/h as the cap, dt = 1 h.  Ages start uniform in
    [0, 120) h so apoptosis (age >= 87 h) runs from the first step (R44); diameters
    start uniform in [10, 14) um so divisions begin early (d_max = 14 um, R43)."""
    name: str
    n: int
    side: float
    d_lo: float
    d_width: float
    steps: int
    max_age0: int = 120
    seed: int = 1


ONCO = OncoConfig("onco", 1_000_000, side_for_fraction(1_000_000, (14.0**4 - 10.0**4) / 16.0, 0.3),
                  10.0, 4.0, 20)

PRESETS = {"cfg1": CFG1, "cfg2": CFG2, "cfg3": CFG3, "cfg4": CFG4, "cfg5": CFG5, "soma": SOMA,
           "onco": ONCO}
