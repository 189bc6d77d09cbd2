"""Golden fixtures for `.tns` ingestion: tucker::load_tns (the UNMODIFIED
reference, oracle/_ref) on a corpus of valid and malformed inputs -> status,
message, ParseError line, and the normalised tensor (dims, coords, values).
TEST INFRASTRUCTURE ONLY; writes tests/golden/tns.npz."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bind import RefLib, ref_load_tns  # noqa: E402


def corpus():
    cases = [
        ("basic", b"# comment\ndims: 4 5 6\n2 3 4 -1.5\n1 1 1 2\n", None),
        ("infer", b"2 3 4 -1.5\n1 1 1 1.0\n", None),
        ("dup", b"1 1 1 1.0\n1 1 1 2.0\n2 1 1 0.5\n", None),
        ("crlf_tabs", b"dims:\t3 3\r\n1\t2  0.25\r\n\r\n3 3 -4e-3\r\n", None),
        ("override", b"1 1 7.0\n2 2 1.0\n", [5, 6]),
        ("override_hdr_ok", b"dims: 9 9\n1 1 7.0\n", [5, 6]),
        ("override_hdr_bad", b"dims: 9 9 9\n1 1 7.0\n", [5, 6]),
        ("header_only", b"dims: 2 2 2\n", None),
        ("empty", b"# nothing\n\n", None),
        ("empty_override", b"", [3, 4]),
        ("empty_header", b"dims:\n1 1 1\n", None),
        ("zero_extent", b"dims: 3 0\n", None),
        ("late_dims", b"1 1 1.0\ndims: 3 3\n", None),
        ("fields", b"1 1 2.5\n1 1 1 1 2.5\n", None),
        ("bad_index", b"1 1 1 1.0\n1 1 nope 2.5\n", None),
        ("neg_index", b"1 -1 1 1.0\n", None),
        ("zero_index", b"0 1 1 2.5\n", None),
        ("big_index", b"4294967297 1 1.0\n", None),
        ("nan", b"1 1 1 nan\n", None),
        ("inf", b"1 1 1 -inf\n", None),
        ("overflow_value", b"1 1 1 1e400\n", None),
        ("plus_value", b"1 1 1 +1.0\n", None),
        ("hex_value", b"1 1 1 0x1p3\n", None),
        ("dot_values", b"1 1 .5\n2 2 5.\n3 3 -0.0\n", None),
        ("one_field", b"7\n", None),
        ("order1", b"3 1.5\n1 2.5\n3 4.0\n", None),
        ("no_newline", b"dims: 2 2\n1 2 3.5", None),
        ("comment_after", b"1 1 1.0\n# 1 1\n   \n2 2 2.0\n", None),
        ("trailing_text", b"1 1 1.0x\n", None),
    ]
    rng = np.random.default_rng(7)
    n = 60000
    c = rng.integers(1, 5000, size=(n, 3))
    v = rng.standard_normal(n)
    big = "".join(f"{a} {b} {d} {x:.17g}\n" for (a, b, d), x in zip(c.tolist(), v.tolist())).encode()
    cases.append(("big", b"dims: 5000 5000 5000\n" + big, None))
    lines = big.split(b"\n")
    lines[n - 1000] = b"17 18 oops 1.0"
    cases.append(("big_late_error", b"\n".join(lines), None))
    lines = big.split(b"\n")
    lines[23456] = b"0 1 1 1.0"
    lines[50000] = b"1 1 1 nan"
    cases.append(("big_first_error", b"\n".join(lines), None))
    return cases


def main():
    lib = RefLib()
    out, names = {}, []
    for name, text, ovr in corpus():
        st, msg, payload, t = ref_load_tns(lib, text, ovr)
        out[f"{name}_text"] = np.frombuffer(text, np.uint8)
        out[f"{name}_override"] = np.asarray(ovr if ovr is not None else [], np.uint64)
        out[f"{name}_status"] = np.array(st)
        out[f"{name}_message"] = np.array(msg)
        out[f"{name}_payload"] = np.array(payload)
        if st == 0:
            c, v = t.export()
            out[f"{name}_dims"] = np.asarray(t.dims, np.uint64)
            out[f"{name}_coords"], out[f"{name}_vals"] = c, v
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "tns.npz"), **out)
    print({n: int(out[f"{n}_status"]) for n in names})


if __name__ == "__main__":
    main()
