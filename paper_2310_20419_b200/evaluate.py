"""Evaluation layer around the GPU search.

Mirrors include/rnnd/eval.hpp and the fvecs/ivecs part of vector_store.hpp:

  EvalRow / mark_pareto / sweep_search / sweep_build /
  report_aod_table / csv_header / csv_row / write_csv      eval.cpp:78-176
  load_fvecs / write_fvecs / load_ivecs / write_ivecs      dataset.cpp:30-132

Searches and builds run on the GPU (rnnd.batch_search / rnnd.build); this
module is the host-side reporting around them, as in the reference.
"""
from __future__ import annotations

import os
import statistics
import struct
import time
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import rnnd as R


# ---------------------------------------------------------------- fvecs

def _read(path: str) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError as e:
        raise R.DataError(f"{path}: cannot open") from e


def _parse_vecs(path: str, buf: bytes, bad_value, value_msg: str) -> Tuple[int, int, np.ndarray]:
    """Record walk shared by both formats (parse_vecs, dataset.cpp:55-78):
    each record is a little-endian int32 dimension followed by that many
    4-byte payloads; every record must have the same positive dimension.  As
    in the reference, records are checked in file order -- a record's header,
    then its values (`bad_value(words) -> bool mask`, `value_msg`), then the
    next record -- and the first problem is reported."""
    if not buf:
        raise R.DataError(f"{path}: empty file")
    if len(buf) < 4:
        raise R.DataError(f"{path}: truncated record header")
    dim = struct.unpack_from("<i", buf, 0)[0]
    if dim <= 0:
        raise R.DataError(f"{path}: non-positive record dimension")
    rec = 4 + 4 * dim
    nrec = len(buf) // rec
    words = np.frombuffer(buf[:nrec * rec], "<u4").reshape(nrec, dim + 1) if nrec else \
        np.zeros((0, dim + 1), "<u4")
    hdr = words[:, 0].view("<i4")
    bad_hdr = np.flatnonzero(hdr != dim)
    first_hdr = int(bad_hdr[0]) if bad_hdr.size else nrec
    bad_val = np.flatnonzero(np.any(bad_value(words[:, 1:]), axis=1))
    first_val = int(bad_val[0]) if bad_val.size else nrec
    if first_val < first_hdr:
        raise R.DataError(f"{path}: {value_msg}")
    if first_hdr < nrec:
        if hdr[first_hdr] <= 0:
            raise R.DataError(f"{path}: non-positive record dimension")
        raise R.DataError(f"{path}: record dimension mismatch")
    rest = len(buf) - nrec * rec
    if rest:
        if rest < 4:
            raise R.DataError(f"{path}: truncated record header")
        d2 = struct.unpack_from("<i", buf, nrec * rec)[0]
        if d2 <= 0:
            raise R.DataError(f"{path}: non-positive record dimension")
        if d2 != dim:
            raise R.DataError(f"{path}: record dimension mismatch")
        raise R.DataError(f"{path}: truncated record payload")
    return nrec, dim, words[:, 1:]


def load_fvecs(path: str) -> R.VectorStore:
    """dataset.cpp:82-95: rejects NaN / Inf."""
    nrec, dim, words = _parse_vecs(
        path, _read(path), lambda w: ~np.isfinite(w.view("<f4")), "non-finite value")
    data = np.ascontiguousarray(words).view("<f4").astype(np.float32)
    return R.VectorStore(data.reshape(nrec, dim))


def write_fvecs(store: R.VectorStore, path: str) -> None:
    if store.n == 0 or store.d == 0:
        raise R.ParamError("write_fvecs: empty store")
    out = np.empty((store.n, store.d + 1), "<u4")
    out[:, 0] = store.d
    out[:, 1:] = np.ascontiguousarray(store.data, "<f4").view("<u4")
    _write(path, out.tobytes())


def load_ivecs(path: str) -> R.GroundTruth:
    """dataset.cpp:109-119: rejects negative ids."""
    nrec, dim, words = _parse_vecs(path, _read(path), lambda w: w.view("<i4") < 0, "negative id")
    return R.GroundTruth(dim, np.ascontiguousarray(words).astype(np.uint32))


def write_ivecs(gt: R.GroundTruth, path: str) -> None:
    if gt.k == 0 or gt.rows() == 0:
        raise R.ParamError("write_ivecs: empty table")
    ids = np.asarray(gt.ids).reshape(-1)
    if ids.size != gt.rows() * gt.k:
        raise R.ParamError("write_ivecs: ragged table")
    out = np.empty((gt.rows(), gt.k + 1), "<u4")
    out[:, 0] = gt.k
    out[:, 1:] = ids.reshape(gt.rows(), gt.k)
    _write(path, out.tobytes())


def _write(path: str, b: bytes) -> None:
    try:
        with open(path, "wb") as f:
            f.write(b)
    except OSError as e:
        raise R.DataError(f"{path}: cannot open for writing") from e


def validate_ids(gt: R.GroundTruth, n: int) -> None:
    """vector_store.hpp:55-56"""
    if np.asarray(gt.ids).size and int(np.max(gt.ids)) >= n:
        raise R.DataError("ground truth id out of range")


# ------------------------------------------------------------------ eval

@dataclass
class EvalRow:
    """eval.hpp:15-30"""

    dataset: str = ""
    n: int = 0
    d: int = 0
    method: str = ""
    S: int = 0
    R: int = 0
    T1: int = 0
    T2: int = 0
    L: int = 0
    K: int = 0
    recall_at_1: float = 0.0
    qps: float = 0.0
    mean_latency_us: float = 0.0
    dist_comps_per_query: float = 0.0
    build_seconds: float = 0.0
    pareto: bool = False


def mark_pareto(rows: List[EvalRow]) -> None:
    """eval.cpp:78-91: strict dominance in (recall@1, qps)."""
    for r in rows:
        r.pareto = True
        for o in rows:
            if o is r:
                continue
            as_good = o.recall_at_1 >= r.recall_at_1 and o.qps >= r.qps
            better = o.recall_at_1 > r.recall_at_1 or o.qps > r.qps
            if as_good and better:
                r.pareto = False
                break


def csv_header() -> str:
    return ("dataset,n,d,method,S,R,T1,T2,L,K,recall_at_1,qps,mean_latency_us,"
            "dist_comps_per_query,build_seconds,pareto")


def csv_row(r: EvalRow) -> str:
    """eval.cpp:160-167 (printf %.6f / %.3f / %.2f formats)."""
    return (f"{r.dataset},{r.n},{r.d},{r.method},{r.S},{r.R},{r.T1},{r.T2},{r.L},{r.K},"
            f"{r.recall_at_1:.6f},{r.qps:.3f},{r.mean_latency_us:.3f},"
            f"{r.dist_comps_per_query:.2f},{r.build_seconds:.3f},{1 if r.pareto else 0}")


def write_csv(rows: List[EvalRow], path: str) -> None:
    _write(path, ("\n".join([csv_header()] + [csv_row(r) for r in rows]) + "\n").encode())


@dataclass
class SweepOptions:
    """eval.hpp:45-51"""

    k: int = 1
    entry_seed: int = R.kDefaultSeed
    threads: int = 0
    reps: int = 3
    warmup: bool = True


@dataclass
class RowContext:
    dataset: str = "synthetic"
    method: str = ""
    S: int = 0
    R: int = 0
    T1: int = 0
    T2: int = 0
    build_seconds: float = 0.0


def _measure_point(g, store, queries, gt, sp, opts: SweepOptions, ctx: RowContext) -> EvalRow:
    """eval.cpp:19-53: warm-up, `reps` timed batches, median wall time."""
    if opts.reps < 1:
        raise R.ParamError("sweep: reps must be >= 1")
    if opts.warmup:
        R.batch_search(g, store, queries, sp)
    walls, res = [], None
    for _ in range(opts.reps):
        t = R.BatchTiming()
        res = R.batch_search(g, store, queries, sp, timing=t)
        walls.append(t.wall_seconds)
    wall = statistics.median(walls)
    comps = sum(r.dist_comps for r in res)
    return EvalRow(dataset=ctx.dataset, n=store.n, d=store.d, method=ctx.method, S=ctx.S,
                   R=ctx.R, T1=ctx.T1, T2=ctx.T2, L=sp.L, K=sp.K,
                   recall_at_1=R.recall_at_1(res, gt, store, queries),
                   qps=queries.n / wall if wall > 0 else 0.0,
                   mean_latency_us=wall * 1e6 / queries.n if queries.n else 0.0,
                   dist_comps_per_query=comps / queries.n if queries.n else 0.0,
                   build_seconds=ctx.build_seconds)


def sweep_search(g, store, queries, gt, Ls: Sequence[int], Ks: Sequence[int],
                 opts: SweepOptions = SweepOptions(), ctx: RowContext = RowContext()
                 ) -> List[EvalRow]:
    """eval.cpp:93-113"""
    if not Ls or not Ks:
        raise R.ParamError("sweep_search: empty L or K list")
    rows = []
    for L in Ls:
        for K in Ks:
            sp = R.SearchParams(L=L, K=K, k=opts.k, seed=opts.entry_seed)
            rows.append(_measure_point(g, store, queries, gt, sp, opts, ctx))
    mark_pareto(rows)
    return rows


def sweep_build(store, queries, gt, t_pairs: Sequence[Tuple[int, int]],
                base_params: R.BuildParams, search_params: R.SearchParams,
                opts: SweepOptions = SweepOptions(), dataset: str = "synthetic") -> List[EvalRow]:
    """eval.cpp:115-142: rebuild per (T1, T2), evaluate at fixed search params."""
    if not t_pairs:
        raise R.ParamError("sweep_build: empty (T1, T2) list")
    rows = []
    for T1, T2 in t_pairs:
        bp = R.BuildParams(S=base_params.S, R=base_params.R, T1=T1, T2=T2,
                           seed=base_params.seed, prune_order=base_params.prune_order)
        st = R.BuildStats()
        g = R.build(store, bp, st)
        ctx = RowContext(dataset, "rnn-descent", bp.S, bp.R, T1, T2, st.seconds)
        rows.append(_measure_point(g, store, queries, gt, search_params, opts, ctx))
    mark_pareto(rows)
    return rows


def report_aod_table(g, caps: Sequence[int]) -> List[Tuple[int, float]]:
    """eval.cpp:144-152: average out-degree per cap, plus uncapped as cap 0."""
    rows = [(c, R.degree_stats(g, c).avg_out) for c in caps]
    if 0 not in caps:
        rows.append((0, R.degree_stats(g, 0).avg_out))
    return rows
