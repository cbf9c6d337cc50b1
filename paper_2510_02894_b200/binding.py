"""In-process replacement of the reference's `shapebind` facade.

Reference: pkg/binding/src/shapebind/__init__.py:94-136 -- `execute(mask,
spacing, backend)` writes a temporary NPY file and runs the CLI in a
subprocess; `dump_arrays(image, mask, out_dir)`.  Here `execute` calls the C
ABI directly (arrays never leave the process; NPY paths are binarized on the
GPU) and keeps the contract: the same 7 keys in the same order, nonzero voxels
are foreground, the same exception types (EngineError, InputError, EmptyRoi,
IoFailure).
"""

from __future__ import annotations

import os
from typing import Dict, Optional, Sequence, Tuple, Union

import numpy as np

from . import errors as _errors
from .features import FEATURE_KEYS

__all__ = ["execute", "dump_arrays", "EngineError", "InputError", "EmptyRoi", "IoFailure"]


class EngineError(RuntimeError):
    """The engine failed (binding __init__.py:43)."""


class InputError(EngineError):
    """The engine rejected the input file or parameters."""


class EmptyRoi(EngineError):
    """The mask contains no foreground voxels."""


class IoFailure(EngineError):
    """An array dump could not be written."""


def _map_errors(fn, *args):
    try:
        return fn(*args)
    except _errors.EmptyRoi as exc:
        raise EmptyRoi(str(exc)) from exc
    except (_errors.NonPositiveSpacing, _errors.MalformedHeader, _errors.UnsupportedDtype,
            _errors.NotThreeDimensional, _errors.TruncatedPayload, _errors.IoFailure,
            ValueError) as exc:
        raise InputError(str(exc)) from exc
    except _errors.ShapeCoreError as exc:
        raise EngineError(str(exc)) from exc


def execute(mask: Union[str, os.PathLike, np.ndarray], spacing: Optional[Sequence[float]] = None,
            backend: str = "auto") -> Dict[str, Union[float, int]]:
    """Feature record of a mask file or 3-D array (binding __init__.py:94-117).
    `backend` is accepted for compatibility; the B200 path is the only one."""
    sp = tuple(spacing) if spacing is not None else (1.0, 1.0, 1.0)
    if isinstance(mask, np.ndarray):
        if mask.ndim != 3:
            raise InputError(f"mask array must be 3-D, got {mask.ndim}-D")
        from .features import calculate_coefficients

        c = _map_errors(calculate_coefficients, mask, sp)
    else:
        from .npy import coefficients_from_npy

        c, _ = _map_errors(coefficients_from_npy, os.fspath(mask), sp)
    record = c.to_dict()
    assert tuple(record) == FEATURE_KEYS
    return record


def dump_arrays(image: np.ndarray, mask: np.ndarray,
                out_dir: Union[str, os.PathLike]) -> Tuple[str, str]:
    """Write (image, mask) as NPY files (binding __init__.py:120-136)."""
    for name, arr in (("image", image), ("mask", mask)):
        if not isinstance(arr, np.ndarray) or arr.ndim != 3:
            raise InputError(f"{name} must be a 3-D array")
    image_path = os.path.join(os.fspath(out_dir), "image.npy")
    mask_path = os.path.join(os.fspath(out_dir), "mask.npy")
    try:
        np.save(image_path, image)
        np.save(mask_path, mask)
    except OSError as exc:
        raise IoFailure(f"cannot write arrays under {out_dir!r}: {exc}") from exc
    return image_path, mask_path
