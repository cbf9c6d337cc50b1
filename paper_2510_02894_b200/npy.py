"""NPY masks: header parsing on the host, binarization on the B200.

Mirrors reference pkg/src/shapecore/volume.py:30-184 (`parse_npy_header`,
`load_npy`, `SUPPORTED_DESCRS`, the error classes) and adds the device path
SURVEY.md 8f #1 asks for: the typed payload is copied to the GPU as is and
binarized there (`sc_calculate_coefficients_raw`), instead of converting on
the host.
"""

from __future__ import annotations

import ast
import ctypes
import struct
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Tuple

import numpy as np

from . import _native
from .errors import (
    IoFailure,
    MalformedHeader,
    NotThreeDimensional,
    TruncatedPayload,
    UnsupportedDtype,
)
from .volume import MaskVolume, _check_spacing

NPY_MAGIC = b"\x93NUMPY"

# descr -> (numpy type, C ABI dtype code); volume.py:34-42
SUPPORTED_DESCRS = {
    "|b1": (np.bool_, 0),
    "|u1": (np.uint8, 1),
    "<i2": (np.int16, 2),
    "<i4": (np.int32, 3),
    "<i8": (np.int64, 4),
    "<f4": (np.float32, 5),
    "<f8": (np.float64, 6),
}


@dataclass(frozen=True)
class NpyHeader:
    version: Tuple[int, int]
    descr: str
    fortran_order: bool
    shape: Tuple[int, ...]

    @property
    def element_count(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64)) if self.shape else 1


def parse_npy_header(fh) -> NpyHeader:
    """Validate the NPY preamble (v1.0 / v2.0), volume.py:104-137 semantics."""
    if fh.read(6) != NPY_MAGIC:
        raise MalformedHeader("not an NPY file (bad magic)")
    ver = fh.read(2)
    if len(ver) != 2:
        raise MalformedHeader("file ends inside the version field")
    if (ver[0], ver[1]) not in ((1, 0), (2, 0)):
        raise MalformedHeader(f"unsupported NPY version {ver[0]}.{ver[1]}")
    size = 2 if ver[0] == 1 else 4
    raw = fh.read(size)
    if len(raw) != size:
        raise MalformedHeader("file ends inside the header-length field")
    (hlen,) = struct.unpack("<H" if size == 2 else "<I", raw)
    text = fh.read(hlen)
    if len(text) != hlen:
        raise MalformedHeader("file ends inside the header dict")
    try:
        meta = ast.literal_eval(text.decode("latin1").strip())
    except (ValueError, SyntaxError) as exc:
        raise MalformedHeader(f"unparseable header dict: {exc}") from exc
    if not isinstance(meta, dict) or not {"descr", "fortran_order", "shape"} <= set(meta):
        raise MalformedHeader(f"header dict missing required keys: {meta!r}")
    if not isinstance(meta["descr"], str):
        raise UnsupportedDtype(f"structured dtypes are not supported: {meta['descr']!r}")
    shape = meta["shape"]
    if not isinstance(shape, tuple) or not all(isinstance(s, int) and s >= 0 for s in shape):
        raise MalformedHeader(f"bad shape entry: {shape!r}")
    if not isinstance(meta["fortran_order"], bool):
        raise MalformedHeader(f"bad fortran_order entry: {meta['fortran_order']!r}")
    return NpyHeader((ver[0], ver[1]), meta["descr"], meta["fortran_order"], shape)


def read_npy_payload(path) -> Tuple[NpyHeader, np.ndarray]:
    """Header + raw typed payload (flat, file order), validated like load_npy."""
    path = Path(path)
    try:
        fh = path.open("rb")
    except OSError as exc:
        raise IoFailure(f"cannot open {path}: {exc}") from exc
    with fh:
        header = parse_npy_header(fh)
        if header.descr not in SUPPORTED_DESCRS:
            raise UnsupportedDtype(f"unsupported element type {header.descr!r}")
        if len(header.shape) != 3:
            raise NotThreeDimensional(f"mask must be 3-D, got shape {header.shape}")
        dtype = np.dtype(SUPPORTED_DESCRS[header.descr][0])
        want = header.element_count * dtype.itemsize
        payload = fh.read(want)
        if len(payload) < want:
            raise TruncatedPayload(f"payload holds {len(payload)} bytes, header declares {want}")
    return header, np.frombuffer(payload, dtype=dtype)


def typed_label(descr: str, label: int):
    """The label as the payload dtype, exactly as numpy's dtype.type(label)."""
    return np.dtype(SUPPORTED_DESCRS[descr][0]).type(label)


def load_npy(path, binarize_label: Optional[int] = None) -> MaskVolume:
    """Host binarization, reference semantics (volume.py:140-184)."""
    header, flat = read_npy_payload(path)
    arr = flat.reshape(header.shape, order="F" if header.fortran_order else "C")
    occ = arr != 0 if binarize_label is None else arr == typed_label(header.descr, binarize_label)
    s0, s1, s2 = header.shape
    return MaskVolume(dims=(s2, s1, s0), spacing=(1.0, 1.0, 1.0),
                      data=np.ascontiguousarray(occ, dtype=np.uint8).reshape(-1),
                      label=binarize_label)


def coefficients_from_npy(path, spacing=(1.0, 1.0, 1.0), label: Optional[int] = None,
                          device: int = 0):
    """File -> coefficients with the binarization on the GPU.  Returns
    (Coefficients, file_read_ms)."""
    from .features import _from_struct
    from .timing import now_ms

    sp = np.asarray(_check_spacing(spacing), dtype=np.float64)
    t0 = now_ms()
    header, flat = read_npy_payload(path)
    t_read = now_ms() - t0
    code = SUPPORTED_DESCRS[header.descr][1]
    has_label = label is not None
    li, lf = 0, 0.0
    if has_label:
        lab = typed_label(header.descr, label)
        if code >= 5:
            lf = float(lab)
        else:
            li = int(lab)
    shape = (ctypes.c_int64 * 3)(*header.shape)
    out = _native.ScCoeffs()
    buf = np.ascontiguousarray(flat)
    rc = _native.load().sc_calculate_coefficients_raw(
        ctypes.c_void_p(buf.ctypes.data), code, shape, int(header.fortran_order), int(has_label),
        li, lf, sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(device),
        ctypes.byref(out))
    _native.raise_for(rc, "sc_calculate_coefficients_raw")
    return _from_struct(out), t_read
