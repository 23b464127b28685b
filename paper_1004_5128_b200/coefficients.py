"""GL history weights ψ(γ, m) generated on the device.

Mirror of /root/reference/pkg/src/fracgrid/coefficients.py.  ``build_table`` runs
the recursion ψ(m) = -ψ(m-1)·(2-γ-m)/m in the ``fg_psi_tables`` kernel with
correctly rounded sub/mul/div (no FMA), so the device table is bitwise equal to
the reference's (coefficients.py:76-92).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import _lib

GAMMA_MIN = 0.0
GAMMA_MAX = 2.0


def _checked_gamma(gamma: float) -> float:
    """coefficients.py:21-27."""
    gamma = float(gamma)
    if not math.isfinite(gamma) or not GAMMA_MIN < gamma < GAMMA_MAX:
        raise ValueError(f"gamma must lie in the open interval ({GAMMA_MIN}, {GAMMA_MAX}), got {gamma!r}")
    return gamma


@dataclass(frozen=True)
class PsiTable:
    """ψ(γ, m) for m = 0..capacity, resident on the device (coefficients.py:54-73).

    ``values`` is a CUDA float64 tensor; treat it as read-only.
    """

    gamma: float
    values: object

    def __post_init__(self) -> None:
        if self.values.dim() != 1 or self.values.numel() < 1:
            raise ValueError("psi table must be a non-empty 1D array")

    @property
    def capacity(self) -> int:
        return int(self.values.numel()) - 1


def build_tables(gammas, n_steps: int, *, device=None):
    """(B, n_steps+1) device tensor of ψ tables, one per γ (batched ensembles)."""
    import torch

    dev = device if device is not None else _lib.require_cuda()
    n_steps = int(n_steps)
    if n_steps < 0:
        raise ValueError(f"n_steps must be >= 0, got {n_steps}")
    g = torch.tensor([_checked_gamma(x) for x in gammas], dtype=torch.float64, device=dev)
    out = torch.empty((g.numel(), n_steps + 1), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().fg_psi_tables(g.data_ptr(), g.numel(), n_steps, n_steps + 1, out.data_ptr(),
                                         _lib.stream_handle()), "fg_psi_tables")
    return out


def build_table(gamma: float, n_steps: int, *, device=None) -> PsiTable:
    """coefficients.py:76-92, on the device."""
    gamma = _checked_gamma(gamma)
    return PsiTable(gamma=gamma, values=build_tables([gamma], n_steps, device=device)[0])


def psi(gamma: float, m: int) -> float:
    """Scalar ψ(γ, m) (coefficients.py:30-51), evaluated by the device recursion."""
    gamma = _checked_gamma(gamma)
    m = int(m)
    if m < 0:
        raise ValueError(f"history offset m must be >= 0, got {m}")
    return float(build_table(gamma, m).values[m].item())


def partial_sum(table: PsiTable, m_max: int) -> float:
    """Σ ψ(0..m_max) (coefficients.py:95-102)."""
    m_max = int(m_max)
    if not 0 <= m_max <= table.capacity:
        raise ValueError(f"m_max must lie in [0, {table.capacity}], got {m_max}")
    return float(table.values[: m_max + 1].cpu().numpy().sum())
