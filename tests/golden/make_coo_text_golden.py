"""Edge-case COO text files and the REFERENCE's load_coo outcome on each
(coo.py:90-148), for tests/test_coo_text.py.  Run in the build container
(imports /root/reference):

    python tests/golden/make_coo_text_golden.py

Writes tests/golden/coo_text/<name>.txt and tests/golden/coo_text/expected.json
({name: {"index_base", "error": [type, message]} or {"dims", "indices",
"values" (float.hex)}}).
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "coo_text")
sys.path.insert(0, "/root/reference/pkg/src")

from sptucker.coo import load_coo  # noqa: E402

CASES = {
    "basic_header": (1, b"# dims: 4 5 6\n1 1 1 1.5\n4 5 6 -2.25\n2 3 4 0\n"),
    "zero_based_noheader": (0, b"0 0 0 1\n3 1 2 2.5e-3\n1 4 0 -7\n"),
    "crlf": (1, b"# dims: 3 3 3\r\n1 2 3 1.0\r\n\r\n3 3 3 2.0\r\n"),
    "lone_cr": (1, b"1 2 3 1.0\r2 2 2 2.0\r\r3 1 1 3.0"),
    "mixed_eol_error": (1, b"1 2 3 1.0\r\n2 2 2 2.0\r3 1 1 x\n"),
    "blank_comment_ws": (1, b"\n   \n# a comment\n\t1\t2  3   4.0  \n#dims: 9 9 9\n  \v2 2 2 5\f\n"),
    "number_forms": (1, b"1_0 +2 007 1_000.5\n1 2 3 .5\n1 2 3 5.\n1 2 3 -0.0\n1 2 3 1E+2\n1 2 3 1e-400\n"
                        b"1 2 3 +1_0e1_0\n1 2 3 4.9406564584124654e-324\n1 2 3 0.1\n1 2 3 1e308\n"),
    "order4": (1, b"1 2 3 4 0.25\n5 6 7 8 -1\n"),
    "order2": (1, b"1 2 3.0\n4 5 6.5\n"),
    "two_headers_last_wins": (1, b"# dims: 2 2 2\n1 1 1 1\n# DIMS: 7 8 9\n2 2 2 2\n"),
    "err_bad_dims": (1, b"1 1 1 1\n# dims: 3 x 3\n2 2 2 2\n"),
    "err_first_line_short": (1, b"# c\n1 2\n1 2 3 4\n"),
    "err_tokens": (1, b"1 2 3 4\n1 2 3\n"),
    "err_unparseable_int": (1, b"1 2 3 4\n1 2.0 3 4\n"),
    "err_unparseable_hex": (1, b"1 2 3 0x10\n"),
    "err_double_underscore": (1, b"1__0 2 3 4\n"),
    "err_leading_underscore": (1, b"1 _2 3 4\n"),
    "err_trailing_underscore": (1, b"1 2 3 4_\n"),
    "err_below_base": (1, b"1 2 3 4\n0 2 3 4\n"),
    "err_negative": (0, b"0 2 3 4\n-1 2 3 4\n"),
    "err_inf": (1, b"1 2 3 inf\n"),
    "err_nan": (1, b"1 2 3 NaN\n"),
    "err_overflow_value": (1, b"1 2 3 1e400\n"),
    "err_empty": (1, b""),
    "err_only_comments": (1, b"# dims: 3 3 3\n\n# nothing\n"),
    "err_dims_len": (1, b"# dims: 3 3\n1 1 1 1\n"),
    "err_overflow_index": (1, b"1 2 3 4\n99999999999999999999 1 1 2\n1 1 1 3\n"),
    "err_overflow_then_format": (1, b"99999999999999999999 1 1 2\n1 1 1 3\n1 1 x 4\n"),
    "err_big_negative": (0, b"1 2 3 4\n-99999999999999999999 1 1 2\n"),
    "err_below_before_nonfinite": (1, b"0 1 1 nan\n"),
    "err_tokens_before_parse": (1, b"1 2 3 4\n1 x 3 4 5\n"),
    "err_dims_header_after_error": (1, b"1 2 3 4\n1 2 3\n# dims: x\n"),
}


def main():
    os.makedirs(OUT, exist_ok=True)
    expected = {}
    for name, (base, data) in CASES.items():
        path = os.path.join(OUT, name + ".txt")
        with open(path, "wb") as fh:
            fh.write(data)
        try:
            t = load_coo(path, index_base=base)
            expected[name] = {"index_base": base, "dims": list(t.dims), "indices": t.indices.tolist(),
                              "values": [float(v).hex() for v in t.values]}
        except Exception as e:  # noqa: BLE001
            expected[name] = {"index_base": base, "error": [type(e).__name__, str(e)]}
        print(name, expected[name].get("error", expected[name].get("dims")))
    with open(os.path.join(OUT, "expected.json"), "w") as fh:
        json.dump(expected, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
