"""`.tns` text parsing (proj/src/sparse_tensor.cpp:97-215), host side.

Parsing text is host work in the reference too; the parsed COO goes straight
to the device builder (SparseTensor).  Error types and messages follow the
reference: ParseError(line) for malformed lines, RangeError for 0-based or
oversized indices, ValueError for non-finite values.
"""
from __future__ import annotations

import io
import math

import numpy as np


def _is_int(tok):
    return tok.isdigit()


def parse_tns(source, dims_override=None):
    from . import ParseError, RangeError, ValueError_

    if isinstance(source, str) and "\n" not in source and not source.strip().startswith(("#", "dims")):
        try:
            fh = open(source)
        except OSError:
            fh = io.StringIO(source)
    elif isinstance(source, str):
        fh = io.StringIO(source)
    else:
        fh = source
    header_dims = []
    coords = []
    values = []
    order = len(dims_override) if dims_override is not None else 0
    observed = None
    saw_content = False
    for line_no, line in enumerate(fh, start=1):
        line = line.rstrip("\n")
        if not line or line[0] == "#" or not line.strip():
            continue
        if not saw_content and line.startswith("dims:"):
            saw_content = True
            toks = line[5:].split()
            if not toks:
                raise ParseError("empty dims header", line_no)
            for t in toks:
                if not _is_int(t):
                    raise ParseError(f"expected an integer index, got '{t}'", line_no)
                d = int(t)
                if d == 0:
                    raise RangeError(f"line {line_no}: extent must be at least 1")
                header_dims.append(d)
            if order and len(header_dims) != order:
                raise ParseError("dims header order does not match override", line_no)
            if not order:
                order = len(header_dims)
            observed = [0] * order
            continue
        saw_content = True
        toks = line.split()
        if not order:
            if len(toks) < 2:
                raise ParseError("entry line needs at least one index and a value", line_no)
            order = len(toks) - 1
            observed = [0] * order
        if len(toks) != order + 1:
            raise ParseError(f"expected {order + 1} fields, got {len(toks)}", line_no)
        if observed is None:
            observed = [0] * order
        row = []
        for m in range(order):
            t = toks[m]
            if not _is_int(t):
                raise ParseError(f"expected an integer index, got '{t}'", line_no)
            idx = int(t)
            if idx < 1:
                raise RangeError(f"line {line_no}: indices are 1-based, got {idx}")
            if idx - 1 > 0xFFFFFFFF:
                raise RangeError(f"line {line_no}: index {idx} too large")
            row.append(idx - 1)
            observed[m] = max(observed[m], idx)
        try:
            v = float(toks[order])
        except ValueError:
            raise ParseError(f"expected a real value, got '{toks[order]}'", line_no)
        if not math.isfinite(v):
            raise ValueError_(f"line {line_no}: non-finite value")
        coords.append(row)
        values.append(v)
    if dims_override is not None:
        dims = list(dims_override)
    elif header_dims:
        dims = header_dims
    elif observed:
        dims = observed
    else:
        raise ParseError("no entries and no dims header; cannot infer tensor order")
    dims = [d if d else 1 for d in dims]
    c = np.asarray(coords, dtype=np.uint32).reshape(-1, len(dims)) if coords else np.zeros((0, len(dims)), np.uint32)
    return dims, c, np.asarray(values, dtype=np.float64)
