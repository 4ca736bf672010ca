"""Seeded synthetic inputs of the BASELINE configs, generated
with the product path (the balanced initial state uses the device
synthesis / Coriolis tendency).  Public benchmark data does not exist for
this path; these stand in for it with the reference's shapes and scalings.
"""

from __future__ import annotations

import dataclasses

import numpy as np

from . import _lib
from .device import pack, to_device, unpack
from .rexi import RexiSetup
from .sphere import SphereConfig, plan_for
from .swe import ModelParams

G = 9.80616


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    trunc: int
    group: str          # "lg" | "l"  (linear REXI group)
    stepper: str        # reference stepper id / description
    dt: float
    n_poles: int
    p0: float = 10.0
    p1: float = 30.0
    steps: int = 1
    phibar: float = 1e4 * G

    @property
    def cfg(self) -> SphereConfig:
        return SphereConfig.for_truncation(self.trunc)

    @property
    def params(self) -> ModelParams:
        return ModelParams(self.phibar, self.cfg)

    @property
    def setup(self) -> RexiSetup:
        return RexiSetup(self.p0, self.p1, self.n_poles)


CONFIGS = {
    "cfg0": Workload("cfg0 lg_rexi T63 N=128", 63, "lg", "lg_rexi", 3600.0, 128),
    "cfg1": Workload("cfg1 l_rexi T128 N=256", 128, "l", "l_rexi", 7200.0, 256),
    "cfg2": Workload("cfg2 lg_rexi_lc_n_etdrk T256 N=256", 256, "lg", "lg_rexi_lc_n_etdrk",
                     1800.0, 256, steps=48),
    "cfg4": Workload("cfg4 l_rexi T1279 N=1024", 1279, "l", "l_rexi", 14400.0, 1024),
    # not a BASELINE config: cfg2's ETD2RK at the north star's largest truncation
    # (dt = 300 s keeps y = dt sqrt(Phibar T(T+1))/a = 18.9 inside the N = 256 contour)
    "etd1279": Workload("lg_rexi_lc_n_etdrk T1279 N=256 (cfg2 setup at T1279)", 1279, "lg",
                        "lg_rexi_lc_n_etdrk", 300.0, 256),
}


@dataclasses.dataclass(frozen=True)
class StiffCase:
    """One cfg3 case: config 2's setup at Phibar = phibar_g * g and dt."""
    phibar_g: float
    dt: float
    y: float            # dt * sqrt(Phibar T (T+1)) / a: the fastest gravity-wave phase
    p1: float
    n_poles: int
    steps: int = 24

    @property
    def phibar(self) -> float:
        return self.phibar_g * G


def stiffness_cases(trunc: int = 256, radius: float = 6.37122e6) -> list:
    """cfg3: Phibar/g in {2000, ..., 18000} (benchmarks.py:240-249)
    x dt in {300, 900, 1800, 3600} s; contour p0 = 10 and the smallest
    power-of-two N with REXI error <= 1e-7 for y = dt sqrt(Phibar T(T+1))/a:
    y <= 15.2 -> (p1 30, N 128); <= 22.7 -> (30, 256); <= 30.5 -> (40, 512);
    <= 45.4 -> (60, 1024); else (80, 2048) (y <= 60.9 at the corner)."""
    table = ((15.2, 30.0, 128), (22.7, 30.0, 256), (30.5, 40.0, 512), (45.4, 60.0, 1024),
             (61.0, 80.0, 2048))
    out = []
    for pg in range(2000, 18001, 2000):
        for dt in (300.0, 900.0, 1800.0, 3600.0):
            y = dt * np.sqrt(pg * G * trunc * (trunc + 1)) / radius
            p1, n = next((p, n) for lim, p, n in table if y <= lim)
            out.append(StiffCase(float(pg), dt, float(y), p1, n))
    return out


def seeded_linear_state(trunc: int, seed: int = 0) -> np.ndarray:
    """cfg0/1/4 input (dense (3, n, n)): amplitudes 1e3, 1e-5, 1e-5 with
    (l+1)^-2 decay; m = 0 real."""
    rng = np.random.default_rng(seed)
    n = trunc + 1
    l = np.arange(n)[:, None]
    m = np.arange(n)[None, :]
    out = np.zeros((3, n, n), dtype=np.complex128)
    for f, amp in enumerate((1e3, 1e-5, 1e-5)):
        c = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * amp / (l + 1.0) ** 2
        c[m > l] = 0.0
        c[:, 0] = c[:, 0].real
        out[f] = c
    return out


def seeded_balanced_state(cfg: SphereConfig, peak: float = 1e-5, seed: int = 0,
                          phibar: float = 1e4 * G) -> np.ndarray:
    """cfg2/3 input: vorticity ~ (l+1)^-1.5 scaled to max|zeta| = peak on the
    grid, zero divergence, phi' in linear balance with the Coriolis term."""
    import torch

    rng = np.random.default_rng(seed)
    n = cfg.trunc + 1
    l = np.arange(n)[:, None]
    m = np.arange(n)[None, :]
    c = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / (l + 1.0) ** 1.5
    c[m > l] = 0.0
    c[:, 0] = c[:, 0].real
    c[0, 0] = 0.0
    plan = plan_for(cfg)
    zmax = float(plan.synthesis_dev(to_device(pack(c[None]), plan.device)).abs().max())
    c = c * (peak / zmax)
    st = np.zeros((3, n, n), dtype=np.complex128)
    st[1] = c
    lc = plan.tendency_dev(_lib.SWX_TEND_LC, to_device(pack(st), plan.device)).cpu().numpy()
    lc = unpack(lc, cfg.trunc)
    kap = (np.arange(n) * (np.arange(n) + 1.0)) / cfg.radius_a**2
    phi = np.zeros((n, n), dtype=np.complex128)
    phi[1:] = -lc[2][1:] / kap[1:, None]
    st[0] = phi
    del torch
    return st
