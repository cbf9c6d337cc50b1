"""shapecore.dispatch compatibility (reference dispatch.py:35-177).

There is no dispatch on the B200 path: north_star rules out multi-backend
dispatch and CPU fallback.  resolve_backend() accepts the reference's request
names and returns a BackendSelection record saying what runs (the B200);
extract_features ignores it."""

import os
from dataclasses import dataclass
from typing import Optional

from paper_2510_02894_b200.pipeline import BACKEND, run_pipeline


@dataclass(frozen=True)
class BackendSelection:
    requested: str
    resolved: str = BACKEND
    worker_count: int = 1
    fallback_reason: Optional[str] = None


def hardware_worker_count() -> int:
    return max(1, os.cpu_count() or 1)


def probe_parallel() -> bool:
    return True


def resolve_backend(requested: str = "auto", workers: Optional[int] = None) -> BackendSelection:
    return BackendSelection(requested=str(requested))


__all__ = ["BackendSelection", "hardware_worker_count", "probe_parallel", "resolve_backend",
           "run_pipeline"]
