"""Host-side evaluation layer: fvecs/ivecs I/O (test_dataset.cpp:37-107),
Pareto marking and CSV format (test_eval.cpp:60-109)."""
import numpy as np
import pytest

from paper_2310_20419_b200 import evaluate as E
from paper_2310_20419_b200 import rnnd as R


def test_fvecs_roundtrip_and_layout(tmp_path):  # test_dataset.cpp:37-48
    p = str(tmp_path / "a.fvecs")
    x = np.array([[1.5, -2.0], [0.0, 3.25]], np.float32)
    E.write_fvecs(R.VectorStore(x), p)
    raw = open(p, "rb").read()
    assert len(raw) == 2 * (4 + 8) and raw[:4] == (2).to_bytes(4, "little")
    back = E.load_fvecs(p)
    assert back.n == 2 and back.d == 2 and np.array_equal(back.data, x)


def test_fvecs_rejects_bad_files(tmp_path):
    p = str(tmp_path / "b.fvecs")
    open(p, "wb").write(b"")
    with pytest.raises(R.DataError, match="empty"):
        E.load_fvecs(p)
    open(p, "wb").write((2).to_bytes(4, "little") + np.float32(1).tobytes())
    with pytest.raises(R.DataError, match="truncated"):
        E.load_fvecs(p)
    open(p, "wb").write((0).to_bytes(4, "little"))
    with pytest.raises(R.DataError, match="non-positive"):
        E.load_fvecs(p)
    rec1 = (1).to_bytes(4, "little") + np.float32(1).tobytes()
    rec2 = (2).to_bytes(4, "little") + np.zeros(2, np.float32).tobytes()
    open(p, "wb").write(rec1 + rec2)
    with pytest.raises(R.DataError, match="mismatch"):
        E.load_fvecs(p)
    open(p, "wb").write((1).to_bytes(4, "little") + np.float32(np.nan).tobytes())
    with pytest.raises(R.DataError, match="non-finite"):
        E.load_fvecs(p)
    with pytest.raises(R.DataError):
        E.load_fvecs(str(tmp_path / "missing.fvecs"))


def test_ivecs_roundtrip_and_validation(tmp_path):  # test_dataset.cpp:50-107
    p = str(tmp_path / "g.ivecs")
    gt = R.GroundTruth(3, np.array([[1, 2, 9], [0, 4, 5]], np.uint32))
    E.write_ivecs(gt, p)
    back = E.load_ivecs(p)
    assert back.k == 3 and np.array_equal(back.ids, gt.ids)
    E.validate_ids(back, 10)
    with pytest.raises(R.DataError):
        E.validate_ids(back, 9)
    open(p, "wb").write((1).to_bytes(4, "little") + b"\xff\xff\xff\xff")
    with pytest.raises(R.DataError, match="negative"):
        E.load_ivecs(p)


def test_pareto_strict_dominance():  # test_eval.cpp:60-83
    rows = [E.EvalRow(recall_at_1=r, qps=q) for r, q in [(0.9, 100), (0.95, 50), (0.9, 120),
                                                          (0.8, 60)]]
    E.mark_pareto(rows)
    assert [r.pareto for r in rows] == [False, True, True, False]
    dup = [E.EvalRow(recall_at_1=0.5, qps=10), E.EvalRow(recall_at_1=0.5, qps=10)]
    E.mark_pareto(dup)
    assert dup[0].pareto and dup[1].pareto


def test_csv_format():  # test_eval.cpp:85-109
    assert E.csv_header() == ("dataset,n,d,method,S,R,T1,T2,L,K,recall_at_1,qps,"
                              "mean_latency_us,dist_comps_per_query,build_seconds,pareto")
    r = E.EvalRow("synthetic", 1000, 32, "rnn-descent", 20, 96, 4, 15, 64, 0, 0.9875,
                  12345.678, 81.0, 420.5, 1.25, True)
    assert E.csv_row(r) == ("synthetic,1000,32,rnn-descent,20,96,4,15,64,0,0.987500,12345.678,"
                            "81.000,420.50,1.250,1")


@pytest.mark.gpu
def test_sweep_search_on_gpu():
    from oracle import oracle as O
    store = R.VectorStore(O.synth_uniform(2000, 8, 3))
    qs = R.VectorStore(O.synth_uniform(100, 8, 4))
    g = R.build(store, R.BuildParams(S=10, R=24, T1=2, T2=4))
    gt = R.brute_force_gt(store, qs, 1)
    rows = E.sweep_search(g, store, qs, gt, [8, 32], [0, 8], E.SweepOptions(reps=1))
    assert len(rows) == 4 and any(r.pareto for r in rows)
    assert rows[1].recall_at_1 <= 1.0 and rows[-1].qps > 0
    aod = E.report_aod_table(g, [4, 8])
    assert aod[-1][0] == 0 and aod[0][1] <= aod[1][1] <= aod[2][1]
