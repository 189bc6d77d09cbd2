"""`.tns` ingestion (proj/src/sparse_tensor.cpp:136-215) through the engine's
native parser (hq_tns_parse, split over host threads) -- same rules, error
types and messages as the reference: ParseError(line) for malformed lines,
RangeError for 0-based / oversized indices or a zero extent, ValueError for
non-finite values.  The parsed COO goes straight to the device builder."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np


def _source_bytes(source):
    """path, text or file object -> (bytes or None, path or None)"""
    if hasattr(source, "read"):
        data = source.read()
        return (data.encode() if isinstance(data, str) else bytes(data)), None
    if isinstance(source, (bytes, bytearray)):
        return bytes(source), None
    if isinstance(source, str) and "\n" not in source and os.path.exists(source):
        return None, source
    return str(source).encode(), None


def _parse_handle(source, dims_override=None):
    from . import _check, load_library
    L = load_library()
    data, path = _source_bytes(source)
    n = 0
    ov = None
    if dims_override is not None:
        ov = np.ascontiguousarray(np.asarray(list(dims_override), dtype=np.uint64))
        n = int(ov.size)
    h = C.c_void_p()
    ovp = ov.ctypes.data if ov is not None else None
    if path is not None:
        _check(L.hq_tns_parse_file(path.encode(), n, ovp, C.byref(h)))
    else:
        _check(L.hq_tns_parse(data, len(data), n, ovp, C.byref(h)))
    return h


def parse_tns(source, dims_override=None):
    """-> (dims, coords nnz x N uint32, values) in file order (host arrays)."""
    from . import _check, load_library
    L = load_library()
    h = _parse_handle(source, dims_override)
    try:
        order, nnz = C.c_int(0), C.c_uint64(0)
        dims = np.zeros(16, np.uint64)
        _check(L.hq_tns_info(h, C.byref(order), dims.ctypes.data, C.byref(nnz)))
        n, z = int(order.value), int(nnz.value)
        nd = len(dims_override) if dims_override is not None else n
        coords = np.empty((z, max(n, 1)), np.uint32)
        vals = np.empty(z, np.float64)
        _check(L.hq_tns_copy(h, coords.ctypes.data, vals.ctypes.data))
        return [int(d) for d in dims[:nd]], coords[:, :n], vals
    finally:
        L.hq_tns_destroy(h)


def load_tns_tensor(source, dims_override=None):
    """Parse and build the device tensor in one step (no host COO copy)."""
    from . import SparseTensor, _check, load_library
    L = load_library()
    h = _parse_handle(source, dims_override)
    try:
        order, nnz = C.c_int(0), C.c_uint64(0)
        dims = np.zeros(16, np.uint64)
        _check(L.hq_tns_info(h, C.byref(order), dims.ctypes.data, C.byref(nnz)))
        nd = len(dims_override) if dims_override is not None else int(order.value)
        t = C.c_void_p()
        _check(L.hq_tns_tensor(h, None, C.byref(t)))
        return SparseTensor([int(d) for d in dims[:nd]], None, None, _handle=t)
    finally:
        L.hq_tns_destroy(h)
