"""Access to the committed reference fixtures (``tests/golden/``).

The fixtures were produced by ``tests/golden/make_golden.py`` from the real
reference package; this module only reads them, so it works on the GPU box where
``/root/reference`` does not exist.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class Golden:
    arrays: dict
    meta: dict

    @classmethod
    def load(cls) -> "Golden":
        with np.load(os.path.join(HERE, "golden.npz")) as z:
            arrays = {k: z[k] for k in z.files}
        with open(os.path.join(HERE, "golden.json")) as fh:
            meta = json.load(fh)
        return cls(arrays, meta)

    def __getitem__(self, key):
        return self.arrays[key]

    # ---- run cases ------------------------------------------------------------
    def run_cases(self, kind=None):
        return [n for n, c in self.meta["cases"].items() if kind is None or c["kind"] == kind]

    def case(self, name):
        return self.meta["cases"][name]

    def initial_field(self, name) -> np.ndarray:
        """Dense (B, *shape) initial field of a case."""
        c = self.case(name)
        if c["kind"] == "nd":
            return self.arrays[f"nd_{name}_u0"]
        key = f"run_{name}_u0"
        if key in self.arrays:
            return self.arrays[key][None]
        u = np.zeros((c["nx"], c["ny"]))
        for j, l, v in c["sources"]:
            u[j, l] = v
        return u[None]

    def expected(self, name):
        """(steps, snaps) with snaps shaped (S, B, *shape)."""
        c = self.case(name)
        if c["kind"] == "nd":
            return self.arrays[f"nd_{name}_steps"], self.arrays[f"nd_{name}_snaps"]
        return self.arrays[f"run_{name}_steps"], self.arrays[f"run_{name}_snaps"][:, None]

    def problem_params(self, name) -> dict:
        """Plain parameters shared by the oracle and the device path."""
        c = self.case(name)
        u0 = self.initial_field(name)
        B = u0.shape[0]
        if c["kind"] == "nd":
            gamma = self.arrays[f"nd_{name}_gamma"]
            dt = self.arrays[f"nd_{name}_dt"]
            reaction = tuple(c["reaction"])
        else:
            gamma = np.full(B, c["gamma"])
            dt = np.full(B, c["dt"])
            reaction = ("linear", c["beta"])
        kind, param = c["strategy"]
        if kind == "adaptive":
            param = int(param)
        return dict(u0=u0, gamma=gamma, dt=dt, alpha=c["alpha"], dx=c["dx"], reaction=reaction,
                    strategy=(kind, param), n_steps=c["n_steps"], snapshot_every=c["snapshot_every"])
