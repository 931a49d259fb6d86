"""Sharded RNN-Descent build: vertex ownership across ranks.

Every rank holds the whole store and owns the lists of a contiguous vertex
range.  Per update pass each rank scans its own lists; the redirects
(w, v, d(v,w)) are records addressed to owner(w) and are exchanged with one
all-to-all.  A reverse phase exchanges three times: reverse proposals to
owner(target), in-edges to owner(target) for in_prune, and the resulting
deletions back to owner(source).  Every step is set-canonical, so the
sharded graph is identical, entry for entry, to the single-device build
(builder.cpp:88-139, :222-251).

The protocol is written against two small interfaces:

* an *engine* per local rank (``DeviceShard``: one ``rnndg_ctx`` with
  ``rnndg_set_partition`` on a GPU; the tests add a CPU restatement), with
  ``random_init / scan / stage / export / import_ / out_prune / counts``;
* a *transport* that moves per-destination record segments:
  ``TorchDistTransport`` (``torch.distributed`` all-to-all: NCCL between GPUs,
  gloo on CPU) or ``LoopbackTransport`` (several ranks in one process).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from . import _lib

X_PENDING, X_PROPOSAL, X_INEDGE, X_DELETE = (_lib.X_PENDING, _lib.X_PROPOSAL, _lib.X_INEDGE,
                                             _lib.X_DELETE)


def ownership_bounds(n: int, world: int) -> List[int]:
    """Contiguous, balanced vertex ranges: rank r owns [b[r], b[r+1])."""
    return [(n * r) // world for r in range(world)] + [n]


# ------------------------------------------------------------- transports

class LoopbackTransport:
    """All ranks live in this process (one engine each): a record sent to
    rank r is simply handed to engine r."""

    def exchange(self, sends):
        """sends[s] = (dst, key, counts[world]) from local rank s, sorted by
        destination.  Returns recvs[r] = (dst, key) for local rank r."""
        import torch
        world = len(sends)
        recvs = []
        for r in range(world):
            ds, ks = [], []
            for dst, key, counts in sends:
                lo = int(sum(counts[:r]))
                hi = lo + int(counts[r])
                if hi > lo:
                    ds.append(dst[lo:hi])
                    ks.append(key[lo:hi])
            if ds:
                recvs.append((torch.cat(ds), torch.cat(ks)))
            else:
                ref = sends[0][0]
                recvs.append((ref[:0], sends[0][1][:0]))
        return recvs

    def allreduce(self, vals: Sequence[np.ndarray]) -> np.ndarray:
        return np.sum(np.stack(vals), axis=0)


class TorchDistTransport:
    """One rank per process; records move with torch.distributed
    all_to_all_single (NCCL for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def exchange(self, sends):
        import torch
        (dst, key, counts), = sends
        dev = dst.device
        sc = torch.tensor([int(c) for c in counts], dtype=torch.int64, device=dev)
        rc = torch.empty_like(sc)
        self.dist.all_to_all_single(rc, sc, group=self.group)
        rcl = [int(x) for x in rc.tolist()]
        scl = [int(x) for x in sc.tolist()]
        rdst = torch.empty(sum(rcl), dtype=dst.dtype, device=dev)
        rkey = torch.empty(sum(rcl), dtype=key.dtype, device=dev)
        self.dist.all_to_all_single(rdst, dst, output_split_sizes=rcl, input_split_sizes=scl,
                                    group=self.group)
        self.dist.all_to_all_single(rkey, key, output_split_sizes=rcl, input_split_sizes=scl,
                                    group=self.group)
        return [(rdst, rkey)]

    def allreduce(self, vals):
        import torch
        (v,), = [vals]
        t = torch.tensor(np.asarray(v, dtype=np.int64))
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()


# ----------------------------------------------------------------- engine

class DeviceShard:
    """One rank's share on a GPU: an rnndg context owning [v_begin, v_end)."""

    def __init__(self, data: np.ndarray, v_begin: int, v_end: int, device: int = 0):
        from .rnnd import Device
        import torch
        self.torch = torch
        self.device = device
        self.dev = Device(device)
        self.v_begin, self.v_end = v_begin, v_end
        self.load(data)
        self._nstaged = 0

    def load(self, data: np.ndarray):
        """(Re)upload the whole store from host memory (H2D) and own
        [v_begin, v_end) again."""
        from .rnnd import VectorStore
        self.store = VectorStore(data)
        self.dev.set_data(self.store)
        self.dev.check(self.dev._L.rnndg_set_partition(self.dev.h, self.v_begin, self.v_end))

    def launches(self) -> int:
        return self.dev.launches()

    def totals(self, reset: bool = False) -> dict:
        """Distance-stage seconds and SURVEY 8(d) units of this shard's scans."""
        s = C.c_double()
        t, a, p = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(self.dev._L.rnndg_shard_totals(self.dev.h, C.byref(s), C.byref(t), C.byref(a),
                                                   C.byref(p), int(reset)))
        return {"scan_seconds": s.value, "touched": t.value, "active_entries": a.value,
                "passes": p.value}

    def _check(self, rc):
        self.dev.check(rc)

    def random_init(self, S: int, seed: int):
        self._check(self.dev._L.rnndg_random_init(self.dev.h, S, seed))

    def scan(self) -> np.ndarray:
        c = _lib.Counts()
        n = C.c_uint64()
        self._check(self.dev._L.rnndg_shard_scan(self.dev.h, C.byref(c), C.byref(n)))
        self._nstaged = n.value
        return np.array([c.removed, 0, c.flag_skips, c.pair_checks], np.int64)

    def stage(self, kind: int):
        n = C.c_uint64()
        self._check(self.dev._L.rnndg_shard_stage(self.dev.h, kind, C.byref(n)))
        self._nstaged = n.value

    def export(self, bounds: Sequence[int]):
        torch = self.torch
        m = self._nstaged
        dst = torch.empty(max(m, 1), dtype=torch.int32, device=f"cuda:{self.device}")
        key = torch.empty(max(m, 1), dtype=torch.int64, device=f"cuda:{self.device}")
        b = np.ascontiguousarray(bounds, np.uint64)
        counts = np.zeros(len(bounds) - 1, np.uint64)
        # the library works on its own stream: memory torch hands out may
        # still be in use by torch-stream work (e.g. the last exchange)
        torch.cuda.current_stream(self.device).synchronize()
        self._check(self.dev._L.rnndg_shard_export(
            self.dev.h, b.ctypes.data_as(_lib.u64p), len(bounds) - 1,
            C.c_void_p(dst.data_ptr()), C.c_void_p(key.data_ptr()),
            counts.ctypes.data_as(_lib.u64p)))
        return dst[:m], key[:m], counts.astype(np.int64)

    def import_(self, kind: int, dst, key, R: int = 0) -> np.ndarray:
        torch = self.torch
        dst = dst.contiguous().to(f"cuda:{self.device}")
        key = key.contiguous().to(f"cuda:{self.device}")
        # the records come from torch-stream work (an NCCL all-to-all, a
        # concatenation): complete it before the library's own stream reads
        # them (without this the import raced the collective)
        torch.cuda.current_stream(self.device).synchronize()
        c = _lib.Counts()
        n = C.c_uint64()
        self._check(self.dev._L.rnndg_shard_import(
            self.dev.h, kind, C.c_void_p(dst.data_ptr() if dst.numel() else 0),
            C.c_void_p(key.data_ptr() if key.numel() else 0), dst.numel(), R, C.byref(c),
            C.byref(n)))
        self._nstaged = n.value
        return np.array([0, c.inserted, 0, 0], np.int64)

    def out_prune(self, R: int):
        self._check(self.dev._L.rnndg_shard_out_prune(self.dev.h, R))

    def graph(self):
        return self.dev.get_graph()


# ----------------------------------------------------------------- driver

@dataclass
class ShardedStats:
    pass_counts: List[np.ndarray] = field(default_factory=list)  # [removed, inserted, skips, checks]

    @property
    def edits(self) -> np.ndarray:
        return np.sum(np.stack(self.pass_counts), axis=0) if self.pass_counts else np.zeros(4)


def _exchange(engines, transport, bounds):
    sends = [e.export(bounds) for e in engines]
    return transport.exchange(sends)


def _in_prune(engines, transport, bounds, R):
    for e in engines:
        e.stage(X_INEDGE)
    recvs = _exchange(engines, transport, bounds)
    for e, (d, k) in zip(engines, recvs):
        e.import_(X_INEDGE, d, k, R)  # stages the deletions
    recvs = _exchange(engines, transport, bounds)
    for e, (d, k) in zip(engines, recvs):
        e.import_(X_DELETE, d, k, R)


def sharded_build(engines, transport, n: int, world: int, S=20, R=96, T1=4, T2=15, seed=42,
                  order: int = 0) -> ShardedStats:
    """rnnd::build (builder.cpp:253-289) over vertex shards.  `engines` are
    this process's ranks (one under torch.distributed, all of them for the
    loopback transport).  Lists come out sorted nearest-first, as after the
    reference's final sort."""
    if n < 2:
        raise ValueError("build: need at least 2 vectors")
    if S < 1 or S > n - 1:
        raise ValueError("build: S out of [1, n-1]")
    if R < 1:
        raise ValueError("build: R must be >= 1")
    if T1 < 1 or T2 < 1:
        raise ValueError("build: T1 and T2 must be >= 1")
    bounds = ownership_bounds(n, world)
    st = ShardedStats()
    local = []  # this process's per-pass partial counts, reduced once at the end
    for e in engines:
        e.random_init(S, seed)
    for t1 in range(1, T1 + 1):
        for _ in range(T2):
            part = [e.scan() for e in engines]
            recvs = _exchange(engines, transport, bounds)
            for i, (e, (d, k)) in enumerate(zip(engines, recvs)):
                part[i] = part[i] + e.import_(X_PENDING, d, k)
            local.append(np.sum(np.stack(part), axis=0))
        if t1 != T1:
            for e in engines:
                e.stage(X_PROPOSAL)
            recvs = _exchange(engines, transport, bounds)
            for e, (d, k) in zip(engines, recvs):
                e.import_(X_PROPOSAL, d, k)
            if order == 0:
                for e in engines:
                    e.out_prune(R)
                _in_prune(engines, transport, bounds, R)
            else:
                _in_prune(engines, transport, bounds, R)
                for e in engines:
                    e.out_prune(R)
    # the counters steer nothing: one all-reduce of the whole [passes, 4]
    # table instead of a host -> device -> host round trip per pass
    total = np.asarray(transport.allreduce([np.stack(local)]))
    st.pass_counts = [total[i] for i in range(total.shape[0])]
    return st


# ------------------------------------------------- one process, C ABI only

class MultiDevice:
    """rnndg_sharded_* (csrc/multi.cu): the same protocol run by the library
    itself over several device contexts in this process -- records move by
    peer copies, no torch.  ``devices`` may repeat (shards sharing a GPU)."""

    def __init__(self, devices: Sequence[int]):
        self._L = _lib.lib()
        self.h = C.c_void_p()
        arr = (C.c_int * len(devices))(*devices)
        rc = self._L.rnndg_sharded_create(C.byref(self.h), arr, len(devices))
        self._check(rc)

    def _check(self, rc):
        if rc != _lib.OK:
            msg = self._L.rnndg_sharded_last_error(self.h).decode() if self.h else "create failed"
            from .rnnd import ParamError, DataError
            if rc == _lib.EPARAM:
                raise ParamError(msg)
            if rc == _lib.EDATA:
                raise DataError(msg)
            raise RuntimeError(msg)

    def close(self):
        if self.h:
            self._L.rnndg_sharded_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_data(self, data: np.ndarray):
        self._data = np.ascontiguousarray(data, np.float32)
        n, d = self._data.shape
        self._check(self._L.rnndg_sharded_set_data(self.h, self._data.ctypes.data_as(_lib.f32p),
                                                   n, d))

    def build(self, S=20, R=96, T1=4, T2=15, seed=42, order=0):
        st = _lib.BuildStatsC()
        self._check(self._L.rnndg_sharded_build(self.h, S, R, T1, T2, seed, order, C.byref(st)))
        npass = C.c_uint32()
        self._check(self._L.rnndg_sharded_pass_counts(self.h, None, 0, C.byref(npass)))
        pc = (_lib.Counts * max(npass.value, 1))()
        self._check(self._L.rnndg_sharded_pass_counts(self.h, pc, npass.value, C.byref(npass)))
        counts = [[c.removed, c.inserted, c.flag_skips, c.pair_checks]
                  for c in pc[:npass.value]]
        return st, counts

    def get_graph(self):
        from .rnnd import CSR
        n, m = C.c_uint64(), C.c_uint64()
        self._check(self._L.rnndg_sharded_graph_size(self.h, C.byref(n), C.byref(m)))
        off = np.empty(n.value + 1, np.uint64)
        ids = np.empty(max(m.value, 1), np.uint32)
        dists = np.empty(max(m.value, 1), np.float32)
        fresh = np.empty(max(m.value, 1), np.uint8)
        self._check(self._L.rnndg_sharded_get_graph(
            self.h, off.ctypes.data_as(_lib.u64p), ids.ctypes.data_as(_lib.u32p),
            dists.ctypes.data_as(_lib.f32p), fresh.ctypes.data_as(_lib.u8p)))
        mm = m.value
        return CSR(off, ids[:mm], dists[:mm], fresh[:mm])
