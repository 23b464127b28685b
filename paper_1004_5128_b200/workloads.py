"""The five BASELINE.json configurations as seeded synthetic inputs.

No dataset is involved: every initial field is generated once on the host with
``numpy.random.default_rng(seed)`` (seeds 0-4 for c1-c5) and the
same fp64 array is fed to the GPU and to the CPU oracle.  Δt is derived from the
stated stability ratio r = α·Δt^γ/Δx², i.e. Δt = (r·Δx²/α)^(1/γ).  Where
BASELINE.json leaves a detail open the choice is recorded here and in DESIGN.md:
adaptive base a = 5 (the reference has no default base), domain [0,1] per axis,
"interior" blob centres drawn from (Δx, 1-Δx), Jacobi pass = mean of the six face
neighbours with the boundary kept at zero, short window L = 500·Δt (floor(L/Δt)
= 500 is asserted).
"""

from __future__ import annotations

import math
from dataclasses import replace

import numpy as np

from .problem import FieldConfig, LinearDecay, Saturating
from .schedule import AdaptiveMemory, FullMemory, ShortMemory

ADAPTIVE_BASE = 5


def dt_for_ratio(r: float, dx: float, gamma: float, alpha: float = 1.0) -> float:
    return (r * dx**2 / alpha) ** (1.0 / gamma)


def _pin(u: np.ndarray) -> np.ndarray:
    for ax in range(u.ndim):
        idx = [slice(None)] * u.ndim
        idx[ax] = 0
        u[tuple(idx)] = 0.0
        idx[ax] = -1
        u[tuple(idx)] = 0.0
    return u


def c1(n_steps: int = 2000) -> FieldConfig:
    """1D, 101 points on [0,1], γ=0.5, r=0.2, no reaction, full memory, snapshot every 100."""
    dx = 0.01
    x = np.arange(101) * dx
    u0 = _pin(np.exp(-((x - 0.5) ** 2) / (2 * 0.05**2)))
    return FieldConfig(initial=u0, dx=dx, gamma=0.5, dt=dt_for_ratio(0.2, dx, 0.5), n_steps=n_steps,
                       strategy=FullMemory(), snapshot_every=100, history_byte_cap=None)


def c2(n_steps: int = 5000, n: int = 256, seed: int = 1) -> FieldConfig:
    """2D 256², γ=0.8, r=0.1, f(u) = -0.1u, Gaussian (σ=0.1, peak 1) + U[0,0.01) noise, adaptive a=5."""
    dx = 1.0 / (n - 1)
    x = np.arange(n) * dx
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = np.exp(-((X - 0.5) ** 2 + (Y - 0.5) ** 2) / (2 * 0.1**2))
    u0 = _pin(u0 + np.random.default_rng(seed).uniform(0.0, 0.01, size=u0.shape))
    return FieldConfig(initial=u0, dx=dx, gamma=0.8, dt=dt_for_ratio(0.1, dx, 0.8), n_steps=n_steps,
                       reaction=LinearDecay(0.1), strategy=AdaptiveMemory(ADAPTIVE_BASE), history_byte_cap=None)


def c3(memory: str = "full", n_steps: int = 4000, n: int = 1024, seed: int = 2) -> FieldConfig:
    """2D 1024², γ=0.6, r=0.1, 64 Gaussian blobs; memory = full | short | adaptive."""
    dx = 1.0 / (n - 1)
    rng = np.random.default_rng(seed)
    x = np.arange(n) * dx
    u0 = np.zeros((n, n))
    for _ in range(64):
        cx, cy = rng.uniform(dx, 1.0 - dx, size=2)
        sig = rng.uniform(0.01, 0.05)
        amp = rng.uniform(0.5, 1.0)
        gx = np.exp(-((x - cx) ** 2) / (2 * sig**2))
        gy = np.exp(-((x - cy) ** 2) / (2 * sig**2))
        u0 += amp * np.outer(gx, gy)
    u0 = _pin(u0)
    dt = dt_for_ratio(0.1, dx, 0.6)
    if memory == "full":
        strat = FullMemory()
    elif memory == "short":
        L = 500 * dt
        assert math.floor(L / dt) == 500
        strat = ShortMemory(L)
    elif memory == "adaptive":
        strat = AdaptiveMemory(ADAPTIVE_BASE)
    else:
        raise ValueError(memory)
    return FieldConfig(initial=u0, dx=dx, gamma=0.6, dt=dt, n_steps=n_steps, strategy=strat, history_byte_cap=None)


def c4(memory: str = "full", n_steps: int = 4000, n: int = 128, seed: int = 3) -> FieldConfig:
    """3D 128³, γ=0.7, r=0.05, f(u) = -0.5u/(0.2+u), U[0,1) smoothed by 3 Jacobi passes."""
    dx = 1.0 / (n - 1)
    v = np.random.default_rng(seed).uniform(0.0, 1.0, size=(n, n, n))
    c = (slice(1, -1),) * 3
    for _ in range(3):
        w = np.zeros_like(v)
        w[c] = (v[2:, 1:-1, 1:-1] + v[:-2, 1:-1, 1:-1] + v[1:-1, 2:, 1:-1] + v[1:-1, :-2, 1:-1]
                + v[1:-1, 1:-1, 2:] + v[1:-1, 1:-1, :-2]) / 6.0
        v = w
    strat = {"full": FullMemory(), "adaptive": AdaptiveMemory(ADAPTIVE_BASE)}[memory]
    return FieldConfig(initial=_pin(v), dx=dx, gamma=0.7, dt=dt_for_ratio(0.05, dx, 0.7), n_steps=n_steps,
                       reaction=Saturating(0.5, 0.2), strategy=strat, history_byte_cap=None)


def c5(n_steps: int = 10000, members: int = 2048, n: int = 512, seed: int = 4) -> FieldConfig:
    """2048 × 1D 512-point members, γ_b ~ U[0.3,0.9], r = 0.2 per member, adaptive a=5."""
    dx = 1.0 / (n - 1)
    rng = np.random.default_rng(seed)
    gammas = rng.uniform(0.3, 0.9, size=members)
    centres = rng.uniform(0.2, 0.8, size=members)
    x = np.arange(n) * dx
    u0 = np.exp(-((x[None, :] - centres[:, None]) ** 2) / (2 * 0.03**2))
    u0[:, 0] = u0[:, -1] = 0.0
    dts = np.array([dt_for_ratio(0.2, dx, float(g)) for g in gammas])
    return FieldConfig(initial=u0, dx=dx, gamma=gammas, dt=dts, n_steps=n_steps,
                       strategy=AdaptiveMemory(ADAPTIVE_BASE), batched=True, history_byte_cap=None)


def subset_members(cfg: FieldConfig, idx) -> FieldConfig:
    """Exact-parity member subset of a batched config (members are independent)."""
    idx = np.asarray(idx)
    return replace(cfg, initial=np.asarray(cfg.initial)[idx], gamma=np.asarray(cfg.gamma)[idx],
                   dt=np.asarray(cfg.dt)[idx])


CONFIGS = {
    "c1": lambda: c1(),
    "c2": lambda: c2(),
    "c3-full": lambda: c3("full"),
    "c3-short": lambda: c3("short"),
    "c3-adaptive": lambda: c3("adaptive"),
    "c4-full": lambda: c4("full"),
    "c4-adaptive": lambda: c4("adaptive"),
    "c5": lambda: c5(),
}
