"""The host-side fvecs/ivecs readers (evaluate.py) report the same result or
the same DataError message as the reference's own loaders (oracle/_ref,
dataset.cpp:55-119) on every malformed case, including which of several
problems comes first in file order."""
import os

import pytest

from oracle import oracle as O
from vecs_cases import FVECS_CASES, IVECS_CASES, make_fvecs, write_raw

HAVE_REF = os.path.exists(O.REF_SO)


def host_result(fn, path):
    from paper_2310_20419_b200 import rnnd as R
    try:
        out = fn(path)
    except R.DataError as e:
        return str(e)
    return out


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("name,records", FVECS_CASES, ids=[c[0] for c in FVECS_CASES])
def test_fvecs_messages_match_reference(tmp_path, name, records):
    from paper_2310_20419_b200 import evaluate as E
    p = str(tmp_path / f"{name}.fvecs")
    make_fvecs(p, name, records)
    ref = O.ref_load_vecs(p)
    got = host_result(lambda q: (lambda s: (s.n, s.d))(E.load_fvecs(q)), p)
    assert got == ref


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("name,records", IVECS_CASES, ids=[c[0] for c in IVECS_CASES])
def test_ivecs_messages_match_reference(tmp_path, name, records):
    from paper_2310_20419_b200 import evaluate as E
    p = str(tmp_path / f"{name}.ivecs")
    write_raw(p, records, "<i4")
    ref = O.ref_load_vecs(p, ivecs=True)
    got = host_result(lambda q: (lambda g: (g.rows(), g.k))(E.load_ivecs(q)), p)
    assert got == ref
