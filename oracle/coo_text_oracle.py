"""TEST INFRASTRUCTURE ONLY -- sequential restatement of the reference's COO
text reader (load_coo, /root/reference/pkg/src/sptucker/coo.py:90-148).

The checker the native multi-threaded parser (libsptk sptk_coo_text_parse,
paper_2204_07104_b200.tensor.load_coo) is compared with on large generated
files; it is itself pinned against the reference's own outputs on the edge
cases in tests/golden/coo_text/ (tests/golden/make_coo_text_golden.py).
Returns (dims, indices int64 [nnz, N], values float64) or raises
ValueError(message) like the reference's CooFormatError.
"""

from __future__ import annotations

import math

import numpy as np


def load_coo(path, index_base: int = 1):
    # coo.py:96-97
    if index_base not in (0, 1):
        raise ValueError("index_base must be 0 or 1")
    header = None
    coords, vals = [], []
    width = None
    with open(path) as fh:  # universal newlines, as coo.py:102
        for lineno, raw in enumerate(fh, start=1):
            text = raw.strip()
            if not text:
                continue
            if text.startswith("#"):  # coo.py:107-114
                body = text[1:].strip()
                if body.lower().startswith("dims:"):
                    try:
                        header = tuple(int(t) for t in body[5:].split())
                    except ValueError:
                        raise ValueError(f"line {lineno}: bad dims header") from None
                continue
            tok = text.split()
            if width is None:  # coo.py:116-121
                width = len(tok)
                if width < 3:
                    raise ValueError(f"line {lineno}: need at least 2 indices and a value")
            if len(tok) != width:  # coo.py:122-125
                raise ValueError(f"line {lineno}: expected {width} tokens, got {len(tok)}")
            try:  # coo.py:126-130
                c = [int(t) for t in tok[:-1]]
                v = float(tok[-1])
            except ValueError:
                raise ValueError(f"line {lineno}: unparseable token") from None
            if any(k < index_base for k in c):  # coo.py:131-134
                raise ValueError(f"line {lineno}: index below base {index_base}")
            if not math.isfinite(v):  # coo.py:135-136
                raise ValueError(f"line {lineno}: non-finite value")
            coords.append([k - index_base for k in c])
            vals.append(v)
    if not coords:  # coo.py:139-140
        raise ValueError("no entries in file")
    idx = np.asarray(coords, dtype=np.int64)
    if header is not None:  # coo.py:142-145
        if len(header) != width - 1:
            raise ValueError("dims header length does not match entry order")
        dims = header
    else:
        dims = tuple(int(m) + 1 for m in idx.max(axis=0))
    return dims, idx, np.asarray(vals, dtype=np.float64)
