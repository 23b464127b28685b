"""Test-side restatement of the reference's deterministic CSV writers.

/root/reference/pkg/src/fracgrid/csvio.py:23-102 (format_float, write_grid_csv,
write_profile_csv, write_trace_csv): shortest round-trip decimal with the
trailing ``.0`` trimmed, ``-0.0`` normalised to ``0``, LF line endings, grid
files one row per fixed l sweeping j.  The reference's ``fracgrid simulate``
(cli.py:246-257) writes grid_final.csv, profile.csv (row l of the source cell),
trace.csv (the source cell over the snapshots) and snapshots/step_NNNNNN.csv.
Pinned byte-for-byte against the real writers in tests/test_csv_artifacts.py.
"""

from __future__ import annotations

import os

import numpy as np


def format_float(x: float) -> str:
    x = float(x)
    if x != x:
        return "nan"
    text = repr(x + 0.0 if x == 0.0 else x)
    return text[:-2] if text.endswith(".0") else text


def _write_lines(path: str, lines) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        for line in lines:
            fh.write(line)
            fh.write("\n")


def write_grid_csv(data, path: str) -> None:
    data = np.asarray(getattr(data, "data", data), dtype=np.float64)
    if data.ndim != 2:
        raise ValueError(f"grid data must be 2D, got shape {data.shape}")
    _write_lines(path, (",".join(format_float(v) for v in row) for row in data.T))


def write_profile_csv(values, path: str) -> None:
    arr = np.asarray(values, dtype=np.float64)
    _write_lines(path, (f"{i},{format_float(v)}" for i, v in enumerate(arr)))


def write_trace_csv(steps, values, path: str) -> None:
    _write_lines(path, (f"{int(s)},{format_float(v)}" for s, v in zip(steps, values)))


def read_grid_csv(path: str) -> np.ndarray:
    with open(path, encoding="utf-8") as fh:
        rows = [[float(c) for c in line.split(",")] for line in fh.read().splitlines() if line]
    return np.array(rows, dtype=np.float64).T


def write_simulate_artifacts(result, config, out_dir: str) -> list[str]:
    """The CSV artifacts of ``fracgrid simulate`` (cli.py:246-257) for one result."""
    from paper_1004_5128_b200.benchmark import source_cell  # benchmark.py:155-160

    os.makedirs(os.path.join(out_dir, "snapshots"), exist_ok=True)
    j, l = source_cell(config)
    names = ["grid_final.csv", "profile.csv", "trace.csv"]
    final = np.asarray(result.final.data)
    write_grid_csv(final, os.path.join(out_dir, names[0]))
    write_profile_csv(final[:, l], os.path.join(out_dir, names[1]))
    steps = [s for s, _ in result.snapshots]
    write_trace_csv(steps, [np.asarray(g.data)[j, l] for _, g in result.snapshots], os.path.join(out_dir, names[2]))
    for s, g in result.snapshots:
        name = os.path.join("snapshots", f"step_{s:06d}.csv")
        write_grid_csv(g, os.path.join(out_dir, name))
        names.append(name)
    return names
