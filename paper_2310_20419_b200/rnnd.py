"""Host-side mirror of the reference `rnnd` API over the B200 C ABI.

Same names, argument meaning, defaults and error classes as the reference
headers (paths relative to /root/reference/proj/include/rnnd):

  VectorStore / GroundTruth          vector_store.hpp:12-33
  NeighborEntry / nearer / AdjacencyGraph   graph.hpp:14-40
  random_init                        graph.hpp:45
  select_nearest / degree_stats      graph.hpp:58-65
  save_index / load_index            graph.hpp:67-75
  PruneOrder / BuildParams / EditCounts / BuildStats   builder.hpp:13-49
  rng_strategy / update_neighbors / add_reverse_edges / build  builder.hpp:51-86
  SearchParams / SearchResult / search / batch_search  search.hpp:13-50
  brute_force_gt                     vector_store.hpp:52-53
  recall_at_1                        eval.hpp:38-43
  ParamError / DataError / kDefaultSeed   common.hpp:12-23

Every compute call runs on the GPU through librnndg.so; there is no CPU
fallback.  Differences from the reference, by design:
  * `threads` is accepted and ignored: the device always runs the deferred,
    canonical update pass (builder.cpp:88-139), which the reference runs for
    every threads > 1.  threads == 1 (the order-dependent serial variant,
    builder.cpp:71-86) is not reproduced.
  * recall_at_k (recall@10) is new; the reference has only recall@1.
"""
from __future__ import annotations

import ctypes as C
import enum
import weakref
import os
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import f32p, ptr, u8p, u32p, u64p

kDefaultSeed = 42


class ParamError(ValueError):
    """Argument outside an operation's documented domain (common.hpp:21-23)."""


class DataError(RuntimeError):
    """Malformed or inconsistent input (common.hpp:16-18)."""


class DeviceError(RuntimeError):
    """CUDA / internal failure (C ABI code RNNDG_EINTERNAL)."""


def _raise(rc: int, msg: str):
    if rc == _lib.OK:
        return
    if rc == _lib.EPARAM:
        raise ParamError(msg)
    if rc == _lib.EDATA:
        raise DataError(msg)
    raise DeviceError(msg)


class PruneOrder(enum.IntEnum):
    kOutThenIn = 0
    kInThenOut = 1


class EntryMode(enum.IntEnum):
    kRandomSample = 0
    kFixedVertex = 1


# ------------------------------------------------------------------ data

@dataclass
class VectorStore:
    """Row-major n x d float32 store (vector_store.hpp:12-20)."""

    data: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.float32))

    def __post_init__(self):
        self.data = np.ascontiguousarray(self.data, dtype=np.float32)
        if self.data.ndim == 1:
            self.data = self.data.reshape(-1, 1)

    @property
    def n(self) -> int:
        return int(self.data.shape[0])

    @property
    def d(self) -> int:
        return int(self.data.shape[1])

    def row(self, i: int) -> np.ndarray:
        return self.data[i]


@dataclass
class GroundTruth:
    """k nearest base ids per query row (vector_store.hpp:22-33)."""

    k: int = 0
    ids: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.uint32))

    def rows(self) -> int:
        return int(self.ids.shape[0]) if self.k else 0

    def row(self, q: int) -> np.ndarray:
        return self.ids[q]


@dataclass
class NeighborEntry:
    id: int
    dist: float
    fresh: bool


def nearer(a: NeighborEntry, b: NeighborEntry) -> bool:
    """Ascending (dist, id) (graph.hpp:21-23)."""
    return a.dist < b.dist if a.dist != b.dist else a.id < b.id


# --------------------------------------------------------------- device

@dataclass
class DeviceStore:
    """A VectorStore resident only on one context's device (Device.load_fvecs)."""

    n: int
    d: int
    device: "Device"


class Device:
    """One rnndg_ctx: a CUDA stream, device buffers, the store and a graph."""

    def __init__(self, device: int = 0):
        self._L = _lib.lib()
        h = C.c_void_p()
        rc = self._L.rnndg_create(C.byref(h), device)
        if rc != _lib.OK:
            _raise(rc, f"rnndg_create(device={device}) failed")
        self.h = h
        self.store_ref = None
        self._owner = None  # weakref: the AdjacencyGraph held in the graph slot

    # A context has one graph slot.  The graph whose newest state lives there
    # is its owner; anything that replaces the slot (another build, a store
    # change, binding another graph) first downloads the owner's state to its
    # host copy, so graphs built on the same Device stay independent values
    # (rnnd::build returns the graph by value, builder.hpp:84-86).
    def _evict(self, keep=None):
        o = self._owner() if self._owner is not None else None
        self._owner = None
        if o is not None and o is not keep and o._dev is self:
            if o._dev_fresh:
                o._csr = self.get_graph()
                o._dev_fresh = False
            o._dev_synced = False  # the slot no longer holds it
        if o is keep and o is not None:
            self._owner = weakref.ref(o)

    def _adopt(self, g: "AdjacencyGraph"):
        g._dev, g._dev_fresh = self, True
        self._owner = weakref.ref(g)

    def close(self):
        if getattr(self, "h", None):
            self._L.rnndg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc != _lib.OK:
            msg = self._L.rnndg_last_error(self.h)
            _raise(rc, msg.decode() if msg else "error")

    def launches(self) -> int:
        return int(self._L.rnndg_kernel_launches(self.h))

    def set_data(self, store: VectorStore):
        if isinstance(store, DeviceStore):  # only its own load puts it on the device
            raise ParamError("no vector data: this device store was replaced or its load failed")
        self._evict()
        self.check(self._L.rnndg_set_data(self.h, ptr(store.data, f32p), store.n, store.d))
        self.store_ref = store

    def load_fvecs(self, path: str) -> "DeviceStore":
        """rnnd::load_fvecs (dataset.cpp:82-95) straight into this context's
        device store: pinned staging, chunked, async H2D (rnndg_load_fvecs).
        The store lives only on the device; pass the returned DeviceStore to
        build() / batch_search() in place of a VectorStore."""
        n = C.c_uint64()
        d = C.c_uint32()
        self._evict()
        self.store_ref = None  # a failed load leaves no store (rnndg_load_fvecs)
        self.check(self._L.rnndg_load_fvecs(self.h, os.fsencode(path), C.byref(n), C.byref(d)))
        ds = DeviceStore(int(n.value), int(d.value), self)
        self.store_ref = ds
        return ds

    def set_graph(self, csr: "CSR", has_distances: bool):
        n = len(csr.offsets) - 1
        self.check(self._L.rnndg_set_graph(
            self.h, n, ptr(csr.offsets, u64p), ptr(csr.ids, u32p),
            ptr(csr.dists, f32p) if has_distances else None, ptr(csr.fresh, u8p)))

    def get_graph(self) -> "CSR":
        n = C.c_uint64()
        m = C.c_uint64()
        self.check(self._L.rnndg_graph_size(self.h, C.byref(n), C.byref(m)))
        mm = m.value
        off = np.empty(n.value + 1, np.uint64)
        ids = np.empty(max(mm, 1), np.uint32)
        dists = np.empty(max(mm, 1), np.float32)
        fresh = np.empty(max(mm, 1), np.uint8)
        self.check(self._L.rnndg_get_graph(self.h, ptr(off, u64p), ptr(ids, u32p),
                                           ptr(dists, f32p), ptr(fresh, u8p)))
        if mm == 0:
            return CSR(off, ids[:0], dists[:0], fresh[:0])
        return CSR(off, ids, dists, fresh)


@dataclass
class CSR:
    offsets: np.ndarray
    ids: np.ndarray
    dists: np.ndarray
    fresh: np.ndarray

    @staticmethod
    def empty(n: int) -> "CSR":
        return CSR(np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32),
                   np.zeros(0, np.float32), np.zeros(0, np.uint8))

    @staticmethod
    def from_lists(lists: Sequence[Sequence[NeighborEntry]]) -> "CSR":
        n = len(lists)
        off = np.zeros(n + 1, np.uint64)
        for u, l in enumerate(lists):
            off[u + 1] = off[u] + len(l)
        flat = [e for l in lists for e in l]
        return CSR(off, np.array([e.id for e in flat], np.uint32),
                   np.array([e.dist for e in flat], np.float32),
                   np.array([1 if e.fresh else 0 for e in flat], np.uint8))


# ---------------------------------------------------------------- graph

class AdjacencyGraph:
    """Per-vertex out-lists (graph.hpp:25-40).

    The authoritative copy lives either on the host (a CSR) or on a device
    context; whichever side is stale is refreshed on demand.
    """

    def __init__(self, n: int = 0):
        self._csr: Optional[CSR] = CSR.empty(n)
        self._dev: Optional[Device] = None
        self._dev_fresh = False  # device holds the newest state
        self._dev_synced = False  # device slot equals the host copy (after a download)
        self.has_distances = True

    # -- construction / views
    @classmethod
    def from_lists(cls, lists, has_distances=True) -> "AdjacencyGraph":
        g = cls(len(lists))
        g._csr = CSR.from_lists(lists)
        g.has_distances = has_distances
        return g

    def _host(self) -> CSR:
        if self._dev_fresh:
            self._csr = self._dev.get_graph()
            self._dev_fresh = False
            self._dev_synced = True  # the slot still holds exactly this state
            self._host_dirty = False
        return self._csr

    def _bind(self, store: VectorStore) -> Device:
        """Device context holding `store` and this graph."""
        if self._dev is None:
            self._dev = Device()
        dev = self._dev
        owner = dev._owner() if dev._owner is not None else None
        if dev.store_ref is not store:
            csr = self._host()
            dev.set_data(store)  # evicts the slot's owner
            dev.set_graph(csr, self.has_distances)
        elif owner is not self or not (self._dev_fresh or self._dev_synced):
            csr = self._host()
            dev._evict(keep=None)
            dev.set_graph(csr, self.has_distances)
        dev._adopt(self)
        return dev

    def size(self) -> int:
        return len(self._host().offsets) - 1

    def __len__(self) -> int:
        return self.size()

    def edge_count(self) -> int:
        return int(self._host().offsets[-1])

    @property
    def csr(self) -> CSR:
        return self._host()

    def list(self, u: int) -> List[NeighborEntry]:
        c = self._host()
        a, b = int(c.offsets[u]), int(c.offsets[u + 1])
        return [NeighborEntry(int(c.ids[j]), float(c.dists[j]), bool(c.fresh[j]))
                for j in range(a, b)]

    @property
    def adj(self) -> List[List[NeighborEntry]]:
        return [self.list(u) for u in range(self.size())]

    def set_lists(self, lists):
        self._csr = CSR.from_lists(lists)
        self._dev_fresh = False
        self._dev_synced = False


# ------------------------------------------------------------- builder

@dataclass
class BuildParams:
    """builder.hpp:15-23"""

    S: int = 20
    R: int = 96
    T1: int = 4
    T2: int = 15
    seed: int = kDefaultSeed
    threads: int = 0
    prune_order: PruneOrder = PruneOrder.kOutThenIn


@dataclass
class EditCounts:
    """builder.hpp:25-38"""

    removed: int = 0
    inserted: int = 0
    flag_skips: int = 0
    pair_checks: int = 0

    def __iadd__(self, o: "EditCounts"):
        self.removed += o.removed
        self.inserted += o.inserted
        self.flag_skips += o.flag_skips
        self.pair_checks += o.pair_checks
        return self

    @staticmethod
    def _from(c: _lib.Counts) -> "EditCounts":
        return EditCounts(int(c.removed), int(c.inserted), int(c.flag_skips),
                          int(c.pair_checks))


@dataclass
class BuildStats:
    """builder.hpp:40-45, plus device timing and roofline inputs."""

    seconds: float = 0.0
    update_passes: int = 0
    reverse_phases: int = 0
    edits: EditCounts = field(default_factory=EditCounts)
    scan_seconds: float = 0.0
    sort_seconds: float = 0.0
    apply_seconds: float = 0.0
    reverse_seconds: float = 0.0
    touched: int = 0
    active_entries: int = 0
    kernel_launches: int = 0
    pass_counts: List[EditCounts] = field(default_factory=list)


BuildProgressFn = Callable[[int, int, EditCounts, float], None]


def random_init(store: VectorStore, S: int, seed: int) -> AdjacencyGraph:
    """graph.cpp:47-63"""
    g = AdjacencyGraph(store.n)
    dev = Device()
    dev.set_data(store)
    dev.check(dev._L.rnndg_random_init(dev.h, S, seed))
    dev._adopt(g)
    return g


def update_neighbors(g: AdjacencyGraph, store: VectorStore, threads: int = 1) -> EditCounts:
    """builder.cpp:214-220 (deferred canonical variant for every `threads`)."""
    if not g.has_distances:
        raise ParamError("update_neighbors: graph has no distances")
    dev = g._bind(store)
    c = _lib.Counts()
    dev.check(dev._L.rnndg_update_pass(dev.h, C.byref(c)))
    return EditCounts._from(c)


def add_reverse_edges(g: AdjacencyGraph, R: int, threads: int = 1,
                      order: PruneOrder = PruneOrder.kOutThenIn,
                      store: Optional[VectorStore] = None) -> None:
    """builder.cpp:222-251.  The device needs the store only for binding; a
    graph already on a device keeps its store."""
    if R < 1:
        raise ParamError("add_reverse_edges: R must be >= 1")
    if not g.has_distances:
        raise ParamError("add_reverse_edges: graph has no distances")
    if g._dev is None or store is not None:
        if store is None:
            store = VectorStore(np.zeros((max(g.size(), 1), 1), np.float32))
        dev = g._bind(store)
    else:
        dev = g._bind(g._dev.store_ref)
    dev.check(dev._L.rnndg_reverse(dev.h, int(R), int(order)))


def build(store: VectorStore, params: BuildParams = BuildParams(),
          stats: Optional[BuildStats] = None,
          progress: Optional[BuildProgressFn] = None,
          device: Optional[Device] = None) -> AdjacencyGraph:
    """builder.cpp:253-289; returns the graph by value (device-resident)."""
    if isinstance(store, DeviceStore):
        device = store.device
    dev = device or Device()
    if dev.store_ref is not store:
        dev.set_data(store)
    st = _lib.BuildStatsC()
    if progress is not None:
        def _cb(t1, T1, outer, elapsed, user):
            progress(int(t1), int(T1), EditCounts._from(outer.contents), float(elapsed))
        cb = _lib.PROGRESS_FN(_cb)
    else:
        cb = _lib.PROGRESS_FN()
    dev._evict()
    dev.check(dev._L.rnndg_build(dev.h, params.S, params.R, params.T1, params.T2,
                                 params.seed, int(params.prune_order), C.byref(st), cb,
                                 None))
    g = AdjacencyGraph(store.n)
    dev._adopt(g)
    if stats is not None:
        stats.seconds = st.seconds
        stats.update_passes = st.update_passes
        stats.reverse_phases = st.reverse_phases
        stats.edits = EditCounts._from(st.edits)
        stats.scan_seconds = st.scan_seconds
        stats.sort_seconds = st.sort_seconds
        stats.apply_seconds = st.apply_seconds
        stats.reverse_seconds = st.reverse_seconds
        stats.touched = st.touched
        stats.active_entries = st.active_entries
        stats.kernel_launches = st.kernel_launches
        npass = params.T1 * params.T2
        arr = (_lib.Counts * npass)()
        dev.check(dev._L.rnndg_pass_counts(dev.h, arr, npass))
        stats.pass_counts = [EditCounts._from(arr[i]) for i in range(npass)]
    return g


@dataclass
class NnDescentParams:
    """nndescent.hpp:12-19"""

    K: int = 64
    sample: int = 10
    iters: int = 10
    pool: int = 0  # 0 selects 2 * K
    seed: int = kDefaultSeed
    threads: int = 0  # accepted, ignored (the device join is deterministic)


class NnDescent:
    """nndescent.hpp:27-47 on the GPU, canonical deferred join: each pass
    snapshots every pool, joins all pairs, then keeps the `cap` nearest
    distinct entries of pool + proposals (include/rnndg.h rnndg_nnd_*).  The
    reference's own join is order-dependent for threads > 1."""

    def __init__(self, store, params: NnDescentParams = NnDescentParams(),
                 device: Optional[Device] = None):
        if isinstance(store, DeviceStore):
            device = store.device
        self.dev = device or Device()
        if self.dev.store_ref is not store:
            self.dev.set_data(store)
        self.store = store
        self.params = params
        self._initialised = False

    def init(self):
        p = self.params
        self.dev._evict()  # the init reuses the graph slot (random_init)
        self.dev.check(self.dev._L.rnndg_nnd_init(self.dev.h, p.K, p.sample, p.iters, p.pool,
                                                  p.seed))
        self._initialised = True

    def join_pass(self) -> int:
        """Returns the number of entries new to the pools."""
        m = C.c_uint64()
        self.dev.check(self.dev._L.rnndg_nnd_pass(self.dev.h, C.byref(m)))
        return int(m.value)

    def pools(self) -> List[List[NeighborEntry]]:
        cap = C.c_uint32()
        self.dev.check(self.dev._L.rnndg_nnd_pools(self.dev.h, C.byref(cap), None, None, None,
                                                   None))
        n, k = self.store.n, int(cap.value)
        cnt = np.zeros(n, np.uint32)
        ids = np.zeros(n * k, np.uint32)
        ds = np.zeros(n * k, np.float32)
        fr = np.zeros(n * k, np.uint8)
        self.dev.check(self.dev._L.rnndg_nnd_pools(self.dev.h, C.byref(cap), ptr(cnt, u32p),
                                                   ptr(ids, u32p), ptr(ds, f32p), ptr(fr, u8p)))
        return [[NeighborEntry(int(ids[u * k + j]), float(ds[u * k + j]), bool(fr[u * k + j]))
                 for j in range(int(cnt[u]))] for u in range(n)]

    def finalize(self) -> "AdjacencyGraph":
        self.dev.check(self.dev._L.rnndg_nnd_finalize(self.dev.h))
        g = AdjacencyGraph(self.store.n)
        self.dev._adopt(g)
        return g


def build_nndescent(store, params: NnDescentParams = NnDescentParams(),
                    stats: Optional[BuildStats] = None,
                    device: Optional[Device] = None) -> "AdjacencyGraph":
    """nndescent.cpp:101-119 on the GPU (canonical deferred join)."""
    if isinstance(store, DeviceStore):
        device = store.device
    dev = device or Device()
    if dev.store_ref is not store:
        dev.set_data(store)
    st = _lib.BuildStatsC()
    dev._evict()
    dev.check(dev._L.rnndg_nnd_build(dev.h, params.K, params.sample, params.iters, params.pool,
                                     params.seed, C.byref(st)))
    g = AdjacencyGraph(store.n)
    dev._adopt(g)
    if stats is not None:
        stats.seconds = st.seconds
        stats.update_passes = st.update_passes
        stats.kernel_launches = st.kernel_launches
    return g


def rng_strategy(store: VectorStore, u: int, candidates: Sequence[NeighborEntry],
                 device: Optional[Device] = None) -> List[NeighborEntry]:
    """builder.cpp:196-212"""
    dev = device or Device()
    if dev.store_ref is not store:
        dev.set_data(store)
    m = len(candidates)
    ids = np.array([e.id for e in candidates], np.uint32)
    ds = np.array([e.dist for e in candidates], np.float32)
    kid = np.zeros(max(m, 1), np.uint32)
    kd = np.zeros(max(m, 1), np.float32)
    nk = C.c_uint32(0)
    dev.check(dev._L.rnndg_rng_strategy(dev.h, u, ptr(ids, u32p), ptr(ds, f32p), m,
                                        ptr(kid, u32p), ptr(kd, f32p), C.byref(nk)))
    return [NeighborEntry(int(kid[i]), float(kd[i]), True) for i in range(nk.value)]


# --------------------------------------------------------------- graph io

def select_nearest(g: AdjacencyGraph, u: int, cap: int) -> List[NeighborEntry]:
    """graph.cpp:65-74 (host view of one list)."""
    out = g.list(u)
    if cap == 0 or len(out) <= cap:
        return out
    if g.has_distances:
        out.sort(key=lambda e: (e.dist, e.id))
    return out[:cap]


@dataclass
class DegreeStats:
    edges: int = 0
    avg_out: float = 0.0
    max_out: int = 0
    max_in: int = 0


def degree_stats(g: AdjacencyGraph, cap: int = 0,
                 store: Optional[VectorStore] = None) -> DegreeStats:
    """graph.cpp:76-100 (summary fields), on the device."""
    dev = g._bind(store if store is not None else
                  (g._dev.store_ref if g._dev is not None else
                   VectorStore(np.zeros((max(g.size(), 1), 1), np.float32))))
    out = np.zeros(3, np.uint64)
    dev.check(dev._L.rnndg_degree_stats(dev.h, cap, ptr(out, u64p)))
    n = g.size()
    return DegreeStats(int(out[0]), float(out[0]) / n if n else 0.0, int(out[1]), int(out[2]))


def index_bytes(g: AdjacencyGraph) -> bytes:
    """The serialized RNND index (graph.cpp:102-126)."""
    if g._dev is not None and g._dev_fresh:
        dev = g._dev
        size = C.c_uint64()
        dev.check(dev._L.rnndg_index_bytes(dev.h, None, C.byref(size)))
        buf = np.zeros(size.value, np.uint8)
        dev.check(dev._L.rnndg_index_bytes(dev.h, ptr(buf, u8p), C.byref(size)))
        return buf.tobytes()
    c = g._host()
    import zlib
    n = len(c.offsets) - 1
    b = bytearray(b"RNND")
    b += np.array([1], "<u4").tobytes() + np.array([n], "<u8").tobytes()
    b += c.offsets.astype("<u8").tobytes() + c.ids.astype("<u4").tobytes()
    b += np.array([zlib.crc32(bytes(b)) & 0xFFFFFFFF], "<u4").tobytes()
    return bytes(b)


def save_index(g: AdjacencyGraph, path: str) -> None:
    try:
        with open(path, "wb") as f:
            f.write(index_bytes(g))
    except OSError as e:
        raise DataError(f"{path}: cannot open for writing") from e


def load_index(path: str) -> AdjacencyGraph:
    """graph.cpp:128-178: validates magic, CRC, version, offsets, ids."""
    import zlib
    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError as e:
        raise DataError(f"{path}: cannot open") from e
    if len(buf) < 4 or buf[:4] != b"RNND":
        raise DataError(f"{path}: bad magic")
    if len(buf) < 16 + 8 + 4:
        raise DataError(f"{path}: truncated header")
    stored = int.from_bytes(buf[-4:], "little")
    if zlib.crc32(buf[:-4]) & 0xFFFFFFFF != stored:
        raise DataError(f"{path}: checksum mismatch")
    if int.from_bytes(buf[4:8], "little") != 1:
        raise DataError(f"{path}: unsupported version")
    n = int.from_bytes(buf[8:16], "little")
    if n == 0:
        raise DataError(f"{path}: empty graph")
    if len(buf) < 16 + (n + 1) * 8 + 4:
        raise DataError(f"{path}: truncated offsets")
    off = np.frombuffer(buf, "<u8", n + 1, 16).astype(np.uint64)
    if off[0] != 0 or np.any(off[1:] < off[:-1]):
        raise DataError(f"{path}: bad offsets")
    m = int(off[-1])
    at = 16 + (n + 1) * 8
    if len(buf) != at + m * 4 + 4:
        raise DataError(f"{path}: size does not match offsets")
    ids = np.frombuffer(buf, "<u4", m, at).astype(np.uint32)
    if m and int(ids.max()) >= n:
        raise DataError(f"{path}: id out of range")
    owner = np.repeat(np.arange(n, dtype=np.uint64), np.diff(off).astype(np.int64))
    if np.any(ids.astype(np.uint64) == owner):
        raise DataError(f"{path}: self-loop")
    pairs = owner * np.uint64(n) + ids.astype(np.uint64)
    if len(np.unique(pairs)) != m:
        raise DataError(f"{path}: duplicate edge")
    g = AdjacencyGraph(n)
    g._csr = CSR(off, ids, np.zeros(m, np.float32), np.zeros(m, np.uint8))
    g.has_distances = False
    return g


# --------------------------------------------------------------- search

@dataclass
class SearchParams:
    """search.hpp:15-23"""

    L: int = 64
    K: int = 0
    k: int = 1
    entry: EntryMode = EntryMode.kRandomSample
    entry_vertex: int = 0
    entry_count: int = 0
    seed: int = kDefaultSeed


@dataclass
class SearchResult:
    ids: np.ndarray
    dists: np.ndarray
    visited: int = 0
    dist_comps: int = 0


@dataclass
class BatchTiming:
    wall_seconds: float = 0.0
    qps: float = 0.0


def _validate_search(g: AdjacencyGraph, store: VectorStore, d: int, p: SearchParams):
    # search.cpp:29-38
    if g.size() == 0:
        raise ParamError("search: empty graph")
    if g.size() != store.n:
        raise ParamError("search: store size mismatch")
    if d != store.d:
        raise ParamError("search: dimension mismatch")
    if p.L < 1:
        raise ParamError("search: L must be >= 1")
    if p.k < 1 or p.k > p.L:
        raise ParamError("search: k out of [1, L]")
    if p.entry == EntryMode.kFixedVertex and p.entry_vertex >= g.size():
        raise ParamError("search: entry vertex out of range")


def batch_search(g: AdjacencyGraph, store: VectorStore, queries: VectorStore,
                 params: SearchParams = SearchParams(), threads: int = 0,
                 timing: Optional[BatchTiming] = None) -> List[SearchResult]:
    """search.cpp:105-132 on the GPU."""
    if queries.n == 0:
        raise ParamError("batch_search: no queries")
    if queries.d != store.d:
        raise ParamError("batch_search: dimension mismatch")
    _validate_search(g, store, queries.d, params)
    ids, dists, vis, comps, wall = _search_raw(g, store, queries.data, params)
    if timing is not None:
        timing.wall_seconds = wall
        timing.qps = queries.n / wall if wall > 0 else 0.0
    out = []
    for q in range(queries.n):
        take = int(np.count_nonzero(ids[q] != 0xFFFFFFFF))
        out.append(SearchResult(ids[q, :take].copy(), dists[q, :take].copy(),
                                int(vis[q]), int(comps[q])))
    return out


def _search_raw(g, store, qdata, p: SearchParams):
    dev = g._bind(store)
    q = np.ascontiguousarray(qdata, np.float32)
    nq = q.shape[0]
    ids = np.zeros((nq, p.k), np.uint32)
    dists = np.zeros((nq, p.k), np.float32)
    vis = np.zeros(nq, np.uint64)
    comps = np.zeros(nq, np.uint64)
    t0 = time.perf_counter()
    dev.check(dev._L.rnndg_search(dev.h, ptr(q, f32p), nq, p.L, p.K, p.k, int(p.entry),
                                  p.entry_vertex, p.entry_count, p.seed, ptr(ids, u32p),
                                  ptr(dists, f32p), ptr(vis, u64p), ptr(comps, u64p)))
    wall = time.perf_counter() - t0
    return ids, dists, vis, comps, wall


def search(g: AdjacencyGraph, store: VectorStore, query, params: SearchParams = SearchParams()
           ) -> SearchResult:
    """search.cpp:98-103"""
    q = np.ascontiguousarray(query, np.float32).reshape(1, -1)
    _validate_search(g, store, q.shape[1], params)
    return batch_search(g, store, VectorStore(q), params)[0]


def brute_force_gt(base: VectorStore, queries: VectorStore, k: int, threads: int = 0,
                   device: Optional[Device] = None) -> GroundTruth:
    """dataset.cpp:175-205 on the GPU (exact, ties to the lower id)."""
    if base.d != queries.d:
        raise DataError("brute_force_gt: dimension mismatch")
    if k < 1 or k > base.n:
        raise ParamError("brute_force_gt: k out of range")
    dev = device or Device()
    if dev.store_ref is not base:
        dev.set_data(base)
    q = np.ascontiguousarray(queries.data, np.float32)
    ids = np.zeros((queries.n, k), np.uint32)
    dev.check(dev._L.rnndg_brute_force(dev.h, ptr(q, f32p), queries.n, k, ptr(ids, u32p)))
    return GroundTruth(k, ids)


# ------------------------------------------------------------------ eval

def l2_sq_rows(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Row-wise squared L2 in the reference's exact summation order
    (metric.hpp:26-45), vectorised over rows with float32 numpy ops (each
    elementwise op is one IEEE rounding, no FMA).  Used by recall only."""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    d = a.shape[1]
    s = np.zeros((a.shape[0], 4), np.float32)
    d4 = d - d % 4
    for i in range(0, d4, 4):
        t = a[:, i:i + 4] - b[:, i:i + 4]
        s += t * t
    tot = (s[:, 0] + s[:, 1]) + (s[:, 2] + s[:, 3])
    for i in range(d4, d):
        t = a[:, i] - b[:, i]
        tot = tot + t * t
    return tot.astype(np.float32)


def recall_at_1(results: List[SearchResult], gt: GroundTruth, base: VectorStore,
                queries: VectorStore) -> float:
    """eval.cpp:57-76: hit when the top id is the true nearest, or its
    distance equals the true nearest distance exactly."""
    if gt.k < 1:
        raise ParamError("recall_at_1: ground truth has no columns")
    if len(results) != gt.rows() or len(results) != queries.n:
        raise ParamError("recall_at_1: result/ground-truth count mismatch")
    if gt.ids.size and int(gt.ids.max()) >= base.n:
        raise DataError("ground truth id out of range")
    truth = gt.ids[:, 0].astype(np.int64)
    tdist = l2_sq_rows(queries.data, base.data[truth])
    hits = 0
    for q, r in enumerate(results):
        if len(r.ids) == 0:
            continue
        if int(r.ids[0]) == int(truth[q]) or np.float32(r.dists[0]) == tdist[q]:
            hits += 1
    return hits / len(results) if results else 0.0


def recall_at_k(results: List[SearchResult], gt: GroundTruth, k: int = 10) -> float:
    """New metric (not in the reference): mean |top-k ∩ GT top-k| / k."""
    tot = 0
    for q, r in enumerate(results):
        tot += len(set(int(i) for i in r.ids[:k]) & set(int(i) for i in gt.ids[q, :k]))
    return tot / (k * len(results)) if results else 0.0
