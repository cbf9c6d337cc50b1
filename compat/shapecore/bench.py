"""shapecore.bench compatibility: BenchRecord / TSV I/O are the B200
package's (reference-compatible both ways); bench_run takes the reference's
signature (bench.py:122-182) and runs every case on the B200."""

from typing import Optional, Sequence

from paper_2510_02894_b200.pipeline import BenchRecord, emit_tsv, parse_tsv, render_tsv, \
    speedup_over_reference
from paper_2510_02894_b200.pipeline import bench_run as _bench_run


def bench_run(dataset_dir: str, spacing: Optional[Sequence[float]] = None,
              backends: Sequence[str] = ("sequential",), repeats: int = 5, warmups: int = 1,
              workers: Optional[int] = None):
    return _bench_run(dataset_dir, spacing, repeats=repeats, warmups=warmups)


def speedup_table(records, baseline_backend: str = "sequential"):
    """Speedups of every backend over `baseline_backend` (bench.py:209-256).
    B200 records carry one backend, so a table needs the baseline's records
    too (e.g. a reference-produced TSV via parse_tsv); MissingBaseline as in
    the reference when they are absent."""
    from paper_2510_02894_b200.errors import MissingBaseline

    base = [r for r in records if r.backend == baseline_backend]
    if not base:
        raise MissingBaseline(f"no records of baseline backend {baseline_backend!r}")
    ours = [r for r in records if r.backend != baseline_backend]
    return speedup_over_reference(ours, base, baseline_backend)

__all__ = ["BenchRecord", "bench_run", "emit_tsv", "parse_tsv", "render_tsv", "speedup_table"]
