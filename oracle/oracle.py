"""ctypes loaders for the CPU checkers -- TEST INFRASTRUCTURE ONLY.

`Oracle` wraps oracle/librnnd_oracle.so (the plain-C restatement of the
reference, rnnd_oracle.c); `Ref` wraps oracle/_ref/librnnd_ref.so (the
UNMODIFIED reference sources compiled by oracle/Makefile).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import this module; the
product (paper_2310_20419_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "librnnd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librnnd_ref.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)


def _p(a, t):
    return a.ctypes.data_as(t)


@dataclass
class CSR:
    """A graph state as CSR arrays (stored list order)."""

    offsets: np.ndarray  # u64 [n+1]
    ids: np.ndarray  # u32 [m]
    dists: np.ndarray  # f32 [m]
    fresh: np.ndarray  # u8 [m]

    @property
    def n(self) -> int:
        return len(self.offsets) - 1

    def canonical(self) -> "CSR":
        """Lists sorted ascending (dist, id): the set-semantics normal form."""
        ids = self.ids.copy()
        dists = self.dists.copy()
        fresh = self.fresh.copy()
        for u in range(self.n):
            a, b = int(self.offsets[u]), int(self.offsets[u + 1])
            if b - a > 1:
                order = np.lexsort((ids[a:b], dists[a:b]))
                ids[a:b] = ids[a:b][order]
                dists[a:b] = dists[a:b][order]
                fresh[a:b] = fresh[a:b][order]
        return CSR(self.offsets.copy(), ids, dists, fresh)

    def same_as(self, other: "CSR") -> bool:
        a, b = self.canonical(), other.canonical()
        return (
            np.array_equal(a.offsets, b.offsets)
            and np.array_equal(a.ids, b.ids)
            and np.array_equal(a.dists.view(np.uint32), b.dists.view(np.uint32))
            and np.array_equal(a.fresh, b.fresh)
        )


def _load_oracle():
    if not os.path.exists(ORACLE_SO):
        raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
    L = C.CDLL(ORACLE_SO)
    L.ro_splitmix_next.restype = C.c_uint64
    L.ro_splitmix_next.argtypes = [u64p]
    L.ro_splitmix_bounded.restype = C.c_uint64
    L.ro_splitmix_bounded.argtypes = [u64p, C.c_uint64]
    L.ro_splitmix_unit_float.restype = C.c_float
    L.ro_splitmix_unit_float.argtypes = [u64p]
    L.ro_mix_seed.restype = C.c_uint64
    L.ro_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
    L.ro_sample_distinct.argtypes = [u64p, C.c_uint32, C.c_uint32, C.c_uint32, u32p]
    L.ro_l2_sq.restype = C.c_float
    L.ro_l2_sq.argtypes = [f32p, f32p, C.c_size_t]
    L.ro_synth_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, f32p]
    L.ro_crc32.restype = C.c_uint32
    L.ro_crc32.argtypes = [u8p, C.c_size_t]
    L.ro_graph_new.restype = C.c_void_p
    L.ro_graph_new.argtypes = [C.c_uint64]
    L.ro_graph_free.argtypes = [C.c_void_p]
    L.ro_graph_edges.restype = C.c_uint64
    L.ro_graph_edges.argtypes = [C.c_void_p]
    L.ro_graph_export.argtypes = [C.c_void_p, u64p, u32p, f32p, u8p]
    L.ro_graph_import.argtypes = [C.c_void_p, u64p, u32p, f32p, u8p]
    L.ro_graph_sort_lists.argtypes = [C.c_void_p]
    L.ro_random_init.restype = C.c_int
    L.ro_random_init.argtypes = [C.c_void_p, f32p, C.c_uint32, C.c_uint32, C.c_uint64]
    L.ro_update_pass.argtypes = [C.c_void_p, f32p, C.c_uint32, u64p]
    L.ro_update_pass_serial.argtypes = [C.c_void_p, f32p, C.c_uint32, u64p]
    L.ro_add_reverse_edges.restype = C.c_int
    L.ro_add_reverse_edges.argtypes = [C.c_void_p, C.c_uint32, C.c_int]
    L.ro_build.restype = C.c_int
    L.ro_build.argtypes = [C.c_void_p, f32p, C.c_uint32, C.c_uint32, C.c_uint32,
                           C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, C.c_int, u64p]
    L.ro_rng_strategy.restype = C.c_int
    L.ro_rng_strategy.argtypes = [f32p, C.c_uint32, C.c_uint32, u32p, f32p,
                                  C.c_uint32, u32p, f32p]
    L.ro_search.restype = C.c_int
    L.ro_search.argtypes = [C.c_void_p, f32p, C.c_uint32, f32p, C.c_uint32,
                            C.c_uint32, C.c_uint32, C.c_int, C.c_uint32, C.c_uint32,
                            C.c_uint64, C.c_int, u32p, f32p, u64p, u64p]
    L.ro_brute_force.argtypes = [f32p, C.c_uint64, C.c_uint32, f32p, C.c_uint64,
                                 C.c_uint32, u32p]
    L.ro_degree_stats.argtypes = [C.c_void_p, C.c_uint32, C.c_int, u64p]
    L.ro_index_bytes.restype = C.c_uint64
    L.ro_index_bytes.argtypes = [C.c_void_p, u8p]
    return L


_ORACLE = None


def lib():
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = _load_oracle()
    return _ORACLE


class OracleGraph:
    """Graph state held by the C oracle."""

    def __init__(self, data: np.ndarray):
        self.data = np.ascontiguousarray(data, dtype=np.float32)
        self.n, self.d = self.data.shape
        self.h = lib().ro_graph_new(self.n)

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _ORACLE is not None:
            _ORACLE.ro_graph_free(h)
            self.h = None

    def _dp(self):
        return _p(self.data, f32p)

    def random_init(self, S: int, seed: int) -> int:
        return lib().ro_random_init(self.h, self._dp(), self.d, S, seed)

    def update_pass(self, serial: bool = False) -> np.ndarray:
        c = np.zeros(4, np.uint64)
        fn = lib().ro_update_pass_serial if serial else lib().ro_update_pass
        fn(self.h, self._dp(), self.d, _p(c, u64p))
        return c

    def add_reverse_edges(self, R: int, order: int = 0) -> int:
        return lib().ro_add_reverse_edges(self.h, R, order)

    def build(self, S=20, R=96, T1=4, T2=15, seed=42, order=0, serial=False):
        pc = np.zeros(T1 * T2 * 4, np.uint64)
        rc = lib().ro_build(self.h, self._dp(), self.d, S, R, T1, T2, seed, order,
                            1 if serial else 0, _p(pc, u64p))
        return rc, pc.reshape(T1 * T2, 4)

    def sort_lists(self):
        lib().ro_graph_sort_lists(self.h)

    def edges(self) -> int:
        return int(lib().ro_graph_edges(self.h))

    def export(self) -> CSR:
        m = self.edges()
        off = np.zeros(self.n + 1, np.uint64)
        ids = np.zeros(max(m, 1), np.uint32)
        dists = np.zeros(max(m, 1), np.float32)
        fresh = np.zeros(max(m, 1), np.uint8)
        lib().ro_graph_export(self.h, _p(off, u64p), _p(ids, u32p), _p(dists, f32p),
                              _p(fresh, u8p))
        return CSR(off, ids[:m], dists[:m], fresh[:m])

    def load(self, g: CSR):
        off = np.ascontiguousarray(g.offsets, np.uint64)
        ids = np.ascontiguousarray(g.ids, np.uint32)
        dists = np.ascontiguousarray(g.dists, np.float32)
        fresh = np.ascontiguousarray(g.fresh, np.uint8)
        lib().ro_graph_import(self.h, _p(off, u64p), _p(ids, u32p), _p(dists, f32p),
                              _p(fresh, u8p))

    # -- NN-Descent baseline (canonical deferred join; rnnd_oracle.c)
    def nnd_init(self, K, sample, iters=10, pool=0, seed=42) -> int:
        _nnd_sigs(lib())
        return lib().ro_nnd_init(self.h, self._dp(), self.d, K, sample, iters, pool, seed)

    def nnd_pass(self, sample, cap) -> int:
        _nnd_sigs(lib())
        return int(lib().ro_nnd_pass(self.h, self._dp(), self.d, sample, cap))

    def nnd_finalize(self, K) -> "OracleGraph":
        _nnd_sigs(lib())
        out = OracleGraph(self.data)
        lib().ro_nnd_finalize(self.h, K, out.h)
        return out

    def index_bytes(self) -> bytes:
        size = lib().ro_index_bytes(self.h, None)
        buf = np.zeros(size, np.uint8)
        lib().ro_index_bytes(self.h, _p(buf, u8p))
        return buf.tobytes()

    def search(self, query, L=64, K=0, k=1, entry_mode=0, entry_vertex=0,
               entry_count=0, seed=42, has_distances=True):
        q = np.ascontiguousarray(query, np.float32)
        ids = np.zeros(k, np.uint32)
        dists = np.zeros(k, np.float32)
        vis = C.c_uint64(0)
        comps = C.c_uint64(0)
        r = lib().ro_search(self.h, self._dp(), self.d, _p(q, f32p), L, K, k,
                            entry_mode, entry_vertex, entry_count, seed,
                            1 if has_distances else 0, _p(ids, u32p), _p(dists, f32p),
                            C.byref(vis), C.byref(comps))
        if r < 0:
            raise ValueError("search: parameter error")
        return ids[:r], dists[:r], vis.value, comps.value

    def degree_stats(self, cap=0, has_distances=True):
        out = np.zeros(3, np.uint64)
        lib().ro_degree_stats(self.h, cap, 1 if has_distances else 0, _p(out, u64p))
        return {"edges": int(out[0]), "max_out": int(out[1]), "max_in": int(out[2])}


def l2_sq(a, b) -> float:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return float(np.float32(lib().ro_l2_sq(_p(a, f32p), _p(b, f32p), a.size)))


def _nnd_sigs(L):
    if getattr(L, "_nnd_sigs", False):
        return
    L.ro_nnd_init.restype = C.c_int
    L.ro_nnd_init.argtypes = [C.c_void_p, f32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                              C.c_uint32, C.c_uint64]
    L.ro_nnd_pass.restype = C.c_uint64
    L.ro_nnd_pass.argtypes = [C.c_void_p, f32p, C.c_uint32, C.c_uint32, C.c_uint32]
    L.ro_nnd_finalize.restype = None
    L.ro_nnd_finalize.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
    L._nnd_sigs = True


def synth_uniform(n, d, seed) -> np.ndarray:
    out = np.zeros((n, d), np.float32)
    lib().ro_synth_uniform(n, d, seed, _p(out, f32p))
    return out


def brute_force(base, queries, k) -> np.ndarray:
    base = np.ascontiguousarray(base, np.float32)
    queries = np.ascontiguousarray(queries, np.float32)
    ids = np.zeros((queries.shape[0], k), np.uint32)
    lib().ro_brute_force(_p(base, f32p), base.shape[0], base.shape[1],
                         _p(queries, f32p), queries.shape[0], k, _p(ids, u32p))
    return ids


def sample_distinct(seed_state: int, n: int, count: int, exclude: int = 0xFFFFFFFF):
    st = C.c_uint64(seed_state)
    out = np.zeros(count, np.uint32)
    lib().ro_sample_distinct(C.byref(st), n, count, exclude, _p(out, u32p))
    return out, st.value


def rng_strategy(data, u, cand_ids, cand_dists):
    data = np.ascontiguousarray(data, np.float32)
    ci = np.ascontiguousarray(cand_ids, np.uint32)
    cd = np.ascontiguousarray(cand_dists, np.float32)
    ki = np.zeros(max(len(ci), 1), np.uint32)
    kd = np.zeros(max(len(ci), 1), np.float32)
    r = lib().ro_rng_strategy(_p(data, f32p), data.shape[1], u, _p(ci, u32p),
                              _p(cd, f32p), len(ci), _p(ki, u32p), _p(kd, f32p))
    if r < 0:
        raise ValueError("rng_strategy: candidate equals u")
    return ki[:r], kd[:r]


# --------------------------------------------------------------- reference

def ref_available() -> bool:
    return os.path.exists(REF_SO)


_REF = None


def ref_lib():
    global _REF
    if _REF is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref`")
        L = C.CDLL(REF_SO)
        L.ref_new.restype = C.c_void_p
        L.ref_new.argtypes = [f32p, C.c_uint64, C.c_uint32]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_max_threads.restype = C.c_int
        L.ref_edges.restype = C.c_uint64
        L.ref_edges.argtypes = [C.c_void_p]
        L.ref_random_init.restype = C.c_int
        L.ref_random_init.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64]
        L.ref_update.restype = C.c_int
        L.ref_update.argtypes = [C.c_void_p, C.c_int, u64p]
        L.ref_reverse.restype = C.c_int
        L.ref_reverse.argtypes = [C.c_void_p, C.c_uint32, C.c_int, C.c_int]
        L.ref_build.restype = C.c_int
        L.ref_build.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                C.c_uint32, C.c_uint64, C.c_int, C.c_int, f64p]
        L.ref_export.argtypes = [C.c_void_p, u64p, u32p, f32p, u8p]
        L.ref_import.argtypes = [C.c_void_p, u64p, u32p, f32p, u8p]
        L.ref_load_vecs.restype = C.c_int
        L.ref_load_vecs.argtypes = [C.c_char_p, C.c_int, u64p, u64p, C.c_char_p, C.c_uint64]
        L.ref_index_bytes.restype = C.c_uint64
        L.ref_index_bytes.argtypes = [C.c_void_p, u8p, C.c_uint64]
        L.ref_batch_search.restype = C.c_double
        L.ref_batch_search.argtypes = [C.c_void_p, f32p, C.c_uint64, C.c_uint32,
                                       C.c_uint32, C.c_uint32, C.c_uint64, C.c_int,
                                       u32p, f32p, u64p, u64p]
        L.ref_brute_force.restype = C.c_int
        L.ref_brute_force.argtypes = [f32p, C.c_uint64, C.c_uint32, f32p, C.c_uint64,
                                      C.c_uint32, C.c_int, u32p]
        _REF = L
    return _REF


class RefGraph:
    """Graph state held by the UNMODIFIED reference library (oracle/_ref)."""

    def __init__(self, data: np.ndarray):
        self.data = np.ascontiguousarray(data, dtype=np.float32)
        self.n, self.d = self.data.shape
        self.h = ref_lib().ref_new(_p(self.data, f32p), self.n, self.d)

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _REF is not None:
            _REF.ref_free(h)
            self.h = None

    def random_init(self, S, seed):
        return ref_lib().ref_random_init(self.h, S, seed)

    def update_pass(self, threads=2):
        c = np.zeros(4, np.uint64)
        rc = ref_lib().ref_update(self.h, threads, _p(c, u64p))
        assert rc == 0
        return c

    def add_reverse_edges(self, R, threads=2, order=0):
        return ref_lib().ref_reverse(self.h, R, threads, order)

    def build(self, S=20, R=96, T1=4, T2=15, seed=42, threads=0, order=0):
        st = np.zeros(7, np.float64)
        rc = ref_lib().ref_build(self.h, S, R, T1, T2, seed, threads, order,
                                 _p(st, f64p))
        return rc, st

    def export(self) -> CSR:
        m = int(ref_lib().ref_edges(self.h))
        off = np.zeros(self.n + 1, np.uint64)
        ids = np.zeros(max(m, 1), np.uint32)
        dists = np.zeros(max(m, 1), np.float32)
        fresh = np.zeros(max(m, 1), np.uint8)
        ref_lib().ref_export(self.h, _p(off, u64p), _p(ids, u32p), _p(dists, f32p),
                             _p(fresh, u8p))
        return CSR(off, ids[:m], dists[:m], fresh[:m])

    def load(self, g: CSR):
        ref_lib().ref_import(self.h, _p(np.ascontiguousarray(g.offsets, np.uint64), u64p),
                             _p(np.ascontiguousarray(g.ids, np.uint32), u32p),
                             _p(np.ascontiguousarray(g.dists, np.float32), f32p),
                             _p(np.ascontiguousarray(g.fresh, np.uint8), u8p))

    def index_bytes(self) -> bytes:
        size = ref_lib().ref_index_bytes(self.h, None, 0)
        buf = np.zeros(size, np.uint8)
        ref_lib().ref_index_bytes(self.h, _p(buf, u8p), size)
        return buf.tobytes()

    def batch_search(self, queries, L=64, K=0, k=1, seed=42, threads=0):
        q = np.ascontiguousarray(queries, np.float32)
        nq = q.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        dists = np.zeros((nq, k), np.float32)
        vis = np.zeros(nq, np.uint64)
        comps = np.zeros(nq, np.uint64)
        wall = ref_lib().ref_batch_search(self.h, _p(q, f32p), nq, L, K, k, seed,
                                          threads, _p(ids, u32p), _p(dists, f32p),
                                          _p(vis, u64p), _p(comps, u64p))
        return ids, dists, vis, comps, wall


def ref_brute_force(base, queries, k, threads=0):
    base = np.ascontiguousarray(base, np.float32)
    queries = np.ascontiguousarray(queries, np.float32)
    ids = np.zeros((queries.shape[0], k), np.uint32)
    ref_lib().ref_brute_force(_p(base, f32p), base.shape[0], base.shape[1],
                              _p(queries, f32p), queries.shape[0], k, threads,
                              _p(ids, u32p))
    return ids


def ref_load_vecs(path: str, ivecs: bool = False):
    """The reference's own load_fvecs / load_ivecs: (n, d) or the DataError
    message (str)."""
    n = np.zeros(1, np.uint64)
    d = np.zeros(1, np.uint64)
    err = C.create_string_buffer(512)
    rc = ref_lib().ref_load_vecs(os.fsencode(path), int(ivecs), _p(n, u64p), _p(d, u64p), err, 512)
    if rc == 0:
        return int(n[0]), int(d[0])
    if rc == 2:
        return err.value.decode()
    raise RuntimeError("reference loader failed")


def ref_nndescent(data, K, sample, iters, pool=0, seed=42):
    """The reference's own NnDescent with threads = 1: (pools after init as
    (cnt, ids, dists) dense n x cap, final graph CSR)."""
    data = np.ascontiguousarray(data, np.float32)
    n, d = data.shape
    # export stride: init fills min(sample, n-1) entries even above the cap
    cap = max(pool if pool else 2 * K, K, min(sample, n - 1))
    L = ref_lib()
    L.ref_nndescent.restype = C.c_int
    L.ref_nndescent.argtypes = [f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, u32p, u32p,
                                f32p, u64p, u32p, f32p]
    pc = np.zeros(n, np.uint32)
    pid = np.zeros(n * cap, np.uint32)
    pd = np.zeros(n * cap, np.float32)
    off = np.zeros(n + 1, np.uint64)
    ids = np.zeros(n * K, np.uint32)
    ds = np.zeros(n * K, np.float32)
    rc = L.ref_nndescent(_p(data, f32p), n, d, K, sample, iters, pool, seed, cap, _p(pc, u32p),
                         _p(pid, u32p), _p(pd, f32p), _p(off, u64p), _p(ids, u32p), _p(ds, f32p))
    if rc:
        return rc
    m = int(off[n])
    return (pc, pid.reshape(n, cap), pd.reshape(n, cap)), CSR(off, ids[:m], ds[:m],
                                                               np.zeros(m, np.uint8))
