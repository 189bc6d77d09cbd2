"""CPU checks of the drop-in boundary: the engine library builds for sm_100a,
loads, and exports every symbol include/hoqri_b200.h declares (no GPU calls)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "hoqri_b200.h")).read()
    return sorted(set(re.findall(r"\b(hq_[a-z_0-9]+)\s*\(", text)))


def test_header_matches_python_binding():
    import paper_2510_16930_b200 as hq
    assert set(declared_symbols()) == set(hq.EXPORTED_SYMBOLS)


def test_engine_exports_every_declared_symbol():
    import paper_2510_16930_b200 as hq
    L = hq.load_library()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.hq_version().decode().startswith("hoqri_b200")


def test_engine_is_sm100a_only():
    import subprocess
    lib = os.path.join(ROOT, "paper_2510_16930_b200", "lib", "libhoqri_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_error_taxonomy_without_gpu():
    """Argument errors are raised before any device work (kernels.cpp:12-22, 90)."""
    import numpy as np
    import paper_2510_16930_b200 as hq
    with pytest.raises(hq.ShapeError):
        hq.SparseTensor([], np.zeros(0, np.uint32), np.zeros(0))
    with pytest.raises(hq.ShapeError):
        hq.SparseTensor([2, 2], np.zeros(3, np.uint32), np.zeros(1))


def test_tns_parser_errors():
    import paper_2510_16930_b200 as hq
    from paper_2510_16930_b200.tns import parse_tns
    dims, c, v = parse_tns("# comment\ndims: 4 5 6\n2 3 4 -1.5\n")
    assert dims == [4, 5, 6] and c.tolist() == [[1, 2, 3]] and v.tolist() == [-1.5]
    assert parse_tns("2 3 4 -1.5\n1 1 1 1.0\n")[0] == [2, 3, 4]
    with pytest.raises(hq.ParseError):
        parse_tns("1 1 2.5\n1 1 1 1 2.5\n")
    try:
        parse_tns("1 1 1 1.0\n1 1 nope 2.5\n")
        raise AssertionError
    except hq.ParseError as e:
        assert e.line_number == 2
    with pytest.raises(hq.RangeError):
        parse_tns("0 1 1 2.5\n")
    with pytest.raises(hq.ValueError_):
        parse_tns("1 1 1 nan\n")
    with pytest.raises(hq.ParseError):
        parse_tns("# nothing\n")
    assert parse_tns("dims: 2 2 2\n")[0] == [2, 2, 2]
