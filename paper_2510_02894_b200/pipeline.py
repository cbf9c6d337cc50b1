"""File -> coefficients pipeline and its measurement surface.

Mirrors reference `run_pipeline` (pkg/src/shapecore/dispatch.py:149-177) and
the benchmark-record half of its harness (bench.py:19-182, 320-394): the same
`BenchRecord` fields, TSV columns and 3-decimal cell format, so TSVs written
here load with the reference's `parse_tsv` and vice versa, and a speedup table
of the B200 path over a reference-produced TSV can be formed
(`speedup_over_reference`).

There is one backend: the B200.  `requested_backend` / `workers` are accepted
for signature compatibility and recorded, never dispatched on.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass
from statistics import median
from typing import List, Optional, Sequence, Tuple

from .errors import IoFailure, NoCasesFound, ShapeCoreError
from .features import ShapeFeatures
from .timing import StageTimings, now_ms

BACKEND = "b200"

RECORD_COLUMNS = ("case_id", "input_bytes", "vertex_count", "backend", "repeat", "file_read_ms",
                  "mesh_ms", "diameters_ms", "total_ms")


@dataclass(frozen=True)
class Selection:
    """What ran (the reference returns a BackendSelection here)."""

    requested: str
    resolved: str = BACKEND
    worker_count: int = 1
    fallback_reason: Optional[str] = None


@dataclass(frozen=True)
class BenchRecord:
    """Same fields as reference bench.BenchRecord (bench.py:48-66)."""

    case_id: str
    input_bytes: int
    vertex_count: int
    backend: str
    repeat_index: int
    file_read_ms: float
    mesh_ms: float
    diameters_ms: float
    total_ms: float
    error: Optional[str] = None


def run_pipeline(mask_path: str, spacing: Optional[Sequence[float]] = None,
                 requested_backend: str = "auto", workers: Optional[int] = None,
                 label: Optional[int] = None, device: int = 0):
    """Load an NPY mask (binarized on the GPU), compute the coefficients.

    Returns (ShapeFeatures, StageTimings, Selection); total_ms spans the whole
    call including the file read, as in dispatch.py:164-177."""
    from .npy import coefficients_from_npy

    t0 = now_ms()
    coeffs, t_read = coefficients_from_npy(mask_path, spacing if spacing is not None
                                           else (1.0, 1.0, 1.0), label=label, device=device)
    total = now_ms() - t0
    feats = ShapeFeatures(coeffs.mesh_volume, coeffs.surface_area, coeffs.max_3d_diameter,
                          coeffs.max_2d_diameter_xy, coeffs.max_2d_diameter_xz,
                          coeffs.max_2d_diameter_yz, coeffs.vertex_count)
    timings = StageTimings(file_read_ms=t_read, mesh_ms=coeffs.mesh_ms,
                           diameters_ms=coeffs.diameters_ms,
                           total_ms=max(total, t_read + coeffs.mesh_ms + coeffs.diameters_ms))
    return feats, timings, Selection(requested=str(requested_backend))


def list_cases(dataset_dir: str) -> List[Tuple[str, str]]:
    """(case_id, path) for every .npy file, lexicographic (bench.py:106-119)."""
    try:
        names = sorted(os.listdir(dataset_dir))
    except OSError as exc:
        raise NoCasesFound(f"cannot list dataset dir {dataset_dir!r}: {exc}") from exc
    cases = [(n[:-4], os.path.join(dataset_dir, n)) for n in names if n.endswith(".npy")]
    if not cases:
        raise NoCasesFound(f"no .npy masks in {dataset_dir!r}")
    return cases


def bench_run(dataset_dir: str, spacing: Optional[Sequence[float]] = None, repeats: int = 5,
              warmups: int = 1, device: int = 0) -> List[BenchRecord]:
    """Every case, `warmups` discarded runs then `repeats` recorded ones; a
    failing case becomes one zeroed record with the error (bench.py:122-182)."""
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    if warmups < 0:
        raise ValueError("warmups must be >= 0")
    out: List[BenchRecord] = []
    for case_id, path in list_cases(dataset_dir):
        try:
            size = os.path.getsize(path)
        except OSError:
            size = 0
        try:
            for _ in range(warmups):
                run_pipeline(path, spacing, device=device)
            for rep in range(repeats):
                f, t, _ = run_pipeline(path, spacing, device=device)
                out.append(BenchRecord(case_id, size, f.vertex_count, BACKEND, rep,
                                       t.file_read_ms, t.mesh_ms, t.diameters_ms, t.total_ms))
        except ShapeCoreError as exc:
            out.append(BenchRecord(case_id, size, 0, BACKEND, 0, 0.0, 0.0, 0.0, 0.0, str(exc)))
    return out


def _cell(v) -> str:
    return f"{v:.3f}" if isinstance(v, float) else str(v)


def render_tsv(records: Sequence[BenchRecord]) -> str:
    """Header + one line per record, floats with 3 decimals (bench.py:324-342)."""
    lines = ["\t".join(RECORD_COLUMNS)]
    for r in records:
        lines.append("\t".join(_cell(v) for v in (
            r.case_id, r.input_bytes, r.vertex_count, r.backend, r.repeat_index,
            r.file_read_ms, r.mesh_ms, r.diameters_ms, r.total_ms)))
    return "\n".join(lines) + "\n"


def emit_tsv(records: Sequence[BenchRecord], path: str) -> None:
    try:
        with open(path, "w", encoding="utf-8", newline="") as fh:
            fh.write(render_tsv(records))
    except OSError as exc:
        raise IoFailure(f"cannot write {path!r}: {exc}") from exc


def parse_tsv(path: str) -> List[BenchRecord]:
    """Read a record TSV (this module's or the reference's) back."""
    try:
        with open(path, encoding="utf-8") as fh:
            rows = [ln.rstrip("\n") for ln in fh if ln.strip()]
    except OSError as exc:
        raise IoFailure(f"cannot read {path!r}: {exc}") from exc
    if not rows or tuple(rows[0].split("\t")) != RECORD_COLUMNS:
        raise ValueError(f"{path!r} is not a benchmark-record TSV")
    recs = []
    for i, ln in enumerate(rows[1:], start=2):
        c = ln.split("\t")
        if len(c) != len(RECORD_COLUMNS):
            raise ValueError(f"{path!r} line {i}: expected {len(RECORD_COLUMNS)} cells")
        recs.append(BenchRecord(c[0], int(c[1]), int(c[2]), c[3], int(c[4]), float(c[5]),
                                float(c[6]), float(c[7]), float(c[8])))
    return recs


@dataclass(frozen=True)
class SpeedupRow:
    case_id: str
    backend: str
    vertex_count: int
    comp_median_ms: float
    total_median_ms: float
    comp_speedup: float
    overall_speedup: float


def speedup_over_reference(ours: Sequence[BenchRecord], reference: Sequence[BenchRecord],
                           baseline_backend: str = "sequential") -> List[SpeedupRow]:
    """Median compute (mesh + diameters) and total speedups of the B200 records
    over reference records of `baseline_backend` (bench.py:205-256 ratios)."""
    def med(recs, key):
        return median([key(r) for r in recs])

    def ok(r):
        return r.error is None and r.total_ms > 0.0

    rows = []
    for case_id in sorted({r.case_id for r in ours if ok(r)}):
        mine = [r for r in ours if r.case_id == case_id and ok(r)]
        base = [r for r in reference if r.case_id == case_id and r.backend == baseline_backend
                and ok(r)]
        if not base:
            continue
        comp = lambda r: r.mesh_ms + r.diameters_ms  # noqa: E731
        c_ours, c_base = med(mine, comp), med(base, comp)
        t_ours, t_base = med(mine, lambda r: r.total_ms), med(base, lambda r: r.total_ms)
        rows.append(SpeedupRow(case_id, BACKEND, mine[0].vertex_count, c_ours, t_ours,
                               c_base / c_ours if c_ours else math.inf,
                               t_base / t_ours if t_ours else math.inf))
    return rows
