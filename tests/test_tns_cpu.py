"""CPU: `.tns` ingestion (hq_tns_parse, threaded native parser) against
tucker::load_tns on a corpus of valid and malformed inputs
(tests/golden/tns.npz, oracle/gen_tns_golden.py): same normalised tensor,
same exception type, message and ParseError line -- including files large
enough to be split over threads, with errors deep inside a chunk."""
import numpy as np
import pytest

import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.tns import parse_tns
from conftest import golden

_G = golden("tns.npz")
_EXC = {4: hq.ParseError, 2: hq.RangeError, 3: hq.ValueError_, 5: hq.CapacityError}


@pytest.mark.parametrize("name", [str(n) for n in _G["names"]])
def test_tns_matches_reference(name, oracle):
    g = _G
    text = g[f"{name}_text"].tobytes()
    ovr = [int(v) for v in g[f"{name}_override"]] or None
    st = int(g[f"{name}_status"])
    if st:
        with pytest.raises(_EXC[st]) as e:
            parse_tns(text, ovr)
        assert str(e.value) == str(g[f"{name}_message"])
        if st == 4:
            assert e.value.line_number == int(g[f"{name}_payload"])
        return
    dims, coords, vals = parse_tns(text, ovr)
    assert dims == [int(d) for d in g[f"{name}_dims"]]
    if vals.size == 0:
        assert g[f"{name}_vals"].size == 0
        return
    oc, ov = oracle.normalize(dims, coords, vals)
    np.testing.assert_array_equal(oc, g[f"{name}_coords"])
    np.testing.assert_array_equal(ov, g[f"{name}_vals"])


def test_tns_file_path(tmp_path, oracle):
    g = _G
    p = tmp_path / "big.tns"
    p.write_bytes(g["big_text"].tobytes())
    dims, coords, vals = parse_tns(str(p))
    oc, ov = oracle.normalize(dims, coords, vals)
    np.testing.assert_array_equal(oc, g["big_coords"])
    np.testing.assert_array_equal(ov, g["big_vals"])
