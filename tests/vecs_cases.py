"""Malformed / edge .fvecs and .ivecs files shared by the loader tests
(parse_vecs, dataset.cpp:55-78; value checks :89, :113)."""
import struct

import numpy as np


def write_raw(path, records, dtype="<f4"):
    with open(path, "wb") as f:
        for dim, vals in records:
            f.write(struct.pack("<i", dim))
            f.write(np.asarray(vals, dtype).tobytes())


FVECS_CASES = [
    ("ok", [(3, [1, 2, 3]), (3, [4, 5, 6])]),
    ("empty", []),
    ("short_header", None),  # 2 bytes
    ("zero_dim", [(0, [])]),
    ("negative_dim", [(-3, [])]),
    ("mismatch", [(3, [1, 2, 3]), (4, [1, 2, 3, 4])]),
    ("truncated_payload", [(3, [1, 2, 3]), (3, [1, 2])]),
    ("nan", [(2, [1, 2]), (2, [np.nan, 0])]),
    ("inf_before_mismatch", [(2, [np.inf, 1]), (3, [1, 2, 3])]),
    ("mismatch_before_nan", [(2, [1, 1]), (3, [1, 2, 3]), (2, [np.nan, 1])]),
    ("trailing_header", None),  # one good record + 3 stray bytes
    ("trailing_bad_dim", [(2, [1, 2]), (0, [])]),
    ("neg_dim_after_good", [(2, [1, 2]), (-1, [])]),
]


def make_fvecs(path, name, records):
    if name == "short_header":
        open(path, "wb").write(b"\x01\x00")
    elif name == "trailing_header":
        write_raw(path, [(2, [1, 2])])
        open(path, "ab").write(b"\x02\x00\x00")
    else:
        write_raw(path, records)


IVECS_CASES = [
    ("ok", [(2, [1, 2]), (2, [3, 4])]),
    ("negative_id", [(2, [1, -2]), (2, [3, 4])]),
    ("neg_before_mismatch", [(2, [-1, 2]), (3, [3, 4, 5])]),
    ("mismatch_before_neg", [(2, [1, 2]), (3, [3, 4, 5]), (2, [-1, 0])]),
]
