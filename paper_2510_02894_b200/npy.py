"""NPY masks: header parsing on the host, binarization on the B200.

Mirrors reference pkg/src/shapecore/volume.py:30-184 (`parse_npy_header`,
`load_npy`, `SUPPORTED_DESCRS`, the error classes) and adds the device path
SURVEY.md 8f #1 asks for: the typed payload's occupied slab (found by one
multi-threaded host scan) crosses PCIe as is, in chunks staged through pinned
buffers, and is binarized on the GPU chunk by chunk
(`sc_calculate_coefficients_raw`, `..._raw_batch`), instead of converting on
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


def _raw_record(path, label: Optional[int]):
    """(sc_raw_mask, payload array kept alive, file_read_ms) of one NPY file."""
    from .timing import now_ms

    t0 = now_ms()
    header, flat = read_npy_payload(path)
    t_read = now_ms() - t0
    code = SUPPORTED_DESCRS[header.descr][1]
    li, lf = 0, 0.0
    if label is not None:
        lab = typed_label(header.descr, label)
        if code >= 5:
            lf = float(lab)
        else:
            li = int(lab)
    buf = np.ascontiguousarray(flat)
    rec = _native.ScRawMask(ctypes.c_void_p(buf.ctypes.data), code, int(header.fortran_order),
                            int(label is not None), li, lf,
                            (ctypes.c_int64 * 3)(*header.shape))
    return rec, buf, t_read


def coefficients_from_npy(path, spacing=(1.0, 1.0, 1.0), label: Optional[int] = None,
                          device: int = 0):
    """File -> coefficients with the binarization on the GPU
    (sc_calculate_coefficients_raw: occupied-slab crop of the typed payload on
    the host, chunked pinned H2D, chunk-wise binarize).  Returns
    (Coefficients, file_read_ms)."""
    from .features import _from_struct

    sp = np.asarray(_check_spacing(spacing), dtype=np.float64)
    rec, buf, t_read = _raw_record(path, label)
    out = _native.ScCoeffs()
    rc = _native.load().sc_calculate_coefficients_raw(
        rec.data, rec.dtype, rec.shape, rec.fortran_order, rec.has_label, rec.label_int,
        rec.label_float, sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(device),
        ctypes.byref(out))
    _native.raise_for(rc, "sc_calculate_coefficients_raw")
    return _from_struct(out), t_read


def coefficients_from_npy_batch(paths, spacings, labels=None, device: int = 0):
    """Many NPY files -> coefficients in one pipelined C call
    (sc_calculate_coefficients_raw_batch).  Returns (records, file_read_ms each)."""
    from .features import _check_spacings, _from_structs

    n = len(paths)
    labels = list(labels) if labels is not None else [None] * n
    recs, keep, reads = [], [], []
    for p, lab in zip(paths, labels):
        r, b, t = _raw_record(p, lab)
        recs.append(r)
        keep.append(b)
        reads.append(t)
    sp = _check_spacings(spacings, n)
    arr = (_native.ScRawMask * n)(*recs)
    outs = (_native.ScCoeffs * n)()
    rc = _native.load().sc_calculate_coefficients_raw_batch(
        arr, sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, int(device), outs)
    _native.raise_for(rc, "sc_calculate_coefficients_raw_batch")
    return _from_structs(outs), reads


def coefficients_from_payloads(payloads, spacings, device: int = 0):
    """In-memory typed payloads [(array (nz, ny, nx) any supported dtype,
    C or Fortran contiguous, label or None)] -> coefficients through
    sc_calculate_coefficients_raw_batch (what a caller that already holds NPY
    payloads, e.g. a file cache, hands the library)."""
    from .features import _check_spacings, _from_structs

    n = len(payloads)
    recs, keep = [], []
    for arr, label in payloads:
        a = np.asarray(arr)
        code = {np.dtype(v[0]): v[1] for v in SUPPORTED_DESCRS.values()}.get(a.dtype)
        if code is None or a.ndim != 3:
            raise UnsupportedDtype(f"unsupported payload {a.dtype} / {a.ndim}-D")
        fortran = bool(a.flags.f_contiguous and not a.flags.c_contiguous)
        if not (a.flags.c_contiguous or fortran):
            a = np.ascontiguousarray(a)
        li, lf = 0, 0.0
        if label is not None:
            lab = a.dtype.type(label)
            if code >= 5:
                lf = float(lab)
            else:
                li = int(lab)
        recs.append(_native.ScRawMask(ctypes.c_void_p(a.ctypes.data), code, int(fortran),
                                      int(label is not None), li, lf,
                                      (ctypes.c_int64 * 3)(*a.shape)))
        keep.append(a)
    sp = _check_spacings(spacings, n)
    arr = (_native.ScRawMask * n)(*recs)
    outs = (_native.ScCoeffs * n)()
    rc = _native.load().sc_calculate_coefficients_raw_batch(
        arr, sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, int(device), outs)
    _native.raise_for(rc, "sc_calculate_coefficients_raw_batch")
    return _from_structs(outs)
