"""CPU restatement of one shard's steps -- TEST INFRASTRUCTURE ONLY.

Implements the engine interface of paper_2310_20419_b200/sharded.py on plain
Python lists with the oracle's exact l2 (oracle/rnnd_oracle.c, which is
pinned to the reference), so the sharding protocol can be run under gloo on
CPU and compared with the unsharded oracle build.  Small inputs only.
"""
import struct

import numpy as np
import torch

from oracle import oracle as O

X_PENDING, X_PROPOSAL, X_INEDGE, X_DELETE = 0, 1, 2, 3


def f32_bits(x: float) -> int:
    return struct.unpack("<I", struct.pack("<f", x))[0]


def bits_f32(b: int) -> float:
    return struct.unpack("<f", struct.pack("<I", b))[0]


def make_key(dist: float, ident: int, fresh: int) -> int:
    return (f32_bits(dist) << 32) | (ident << 1) | (fresh & 1)


def split_key(k: int):
    return bits_f32(k >> 32), (k & 0xFFFFFFFF) >> 1, k & 1


class CpuShard:
    def __init__(self, data: np.ndarray, v_begin: int, v_end: int):
        self.x = np.ascontiguousarray(data, np.float32)
        self.v0, self.v1 = v_begin, v_end
        self.lists = {u: [] for u in range(v_begin, v_end)}  # u -> [(id, dist, fresh)]
        self.staged = []  # [(dst, key)]

    def _l2(self, a: int, b: int) -> float:
        return O.l2_sq(self.x[a], self.x[b])

    def random_init(self, S, seed):
        g = O.OracleGraph(self.x)
        assert g.random_init(S, seed) == 0
        c = g.export()
        for u in range(self.v0, self.v1):
            a, b = int(c.offsets[u]), int(c.offsets[u + 1])
            self.lists[u] = [(int(c.ids[j]), float(c.dists[j]), int(c.fresh[j])) for j in range(a, b)]

    def scan(self):
        removed = skips = checks = 0
        self.staged = []
        for u in range(self.v0, self.v1):  # scan_vertex, builder.cpp:45-69
            cand = sorted(self.lists[u], key=lambda e: (np.float32(e[1]), e[0]))
            kept = []
            for v in cand:
                keep = True
                for w in kept:
                    if not v[2] and not w[2]:
                        skips += 1
                        continue
                    checks += 1
                    d = self._l2(v[0], w[0])
                    if np.float32(v[1]) >= np.float32(d):
                        keep = False
                        removed += 1
                        self.staged.append((w[0], make_key(d, v[0], 1)))
                        break
                if keep:
                    kept.append(v)
            self.lists[u] = [(e[0], e[1], 0) for e in kept]
        return np.array([removed, 0, skips, checks], np.int64)

    def stage(self, kind):
        fresh = 1 if kind == X_PROPOSAL else 0
        self.staged = [(e[0], make_key(e[1], u, fresh)) for u, l in self.lists.items() for e in l]

    def export(self, bounds):
        recs = sorted(self.staged)
        dst = torch.tensor([r[0] for r in recs], dtype=torch.int32)
        key = torch.tensor(np.array([r[1] for r in recs], np.uint64).view(np.int64), dtype=torch.int64)
        counts = [sum(1 for r in recs if bounds[p] <= r[0] < bounds[p + 1])
                  for p in range(len(bounds) - 1)]
        return dst, key, np.array(counts, np.int64)

    def import_(self, kind, dst, key, R=0):
        recs = list(zip(dst.tolist(), key.numpy().view(np.uint64).tolist()))
        inserted = 0
        if kind in (X_PENDING, X_PROPOSAL):
            # sort + unique, append-if-absent (builder.cpp:117-136, :230-243)
            seen = set()
            for d, k in sorted(recs, key=lambda r: (r[0], split_key(r[1])[1])):
                dist, ident, fr = split_key(k)
                if (d, ident) in seen:
                    continue
                seen.add((d, ident))
                if all(e[0] != ident for e in self.lists[d]):
                    self.lists[d].append((ident, dist, 1))
                    inserted += 1
            self.staged = []
        elif kind == X_INEDGE:
            # in_prune, builder.cpp:162-176, at the target's owner
            by_t = {}
            for d, k in recs:
                by_t.setdefault(d, []).append(split_key(k))
            self.staged = []
            for t, ins in by_t.items():
                ins.sort(key=lambda r: (np.float32(r[0]), r[1]))
                for dist, src, _ in ins[R:]:
                    self.staged.append((src, make_key(dist, t, 0)))
        else:  # X_DELETE at the source's owner
            for s, k in recs:
                _, t, _ = split_key(k)
                self.lists[s] = [e for e in self.lists[s] if e[0] != t]
            self.staged = []
        return np.array([0, inserted if kind == X_PENDING else 0, 0, 0], np.int64)

    def out_prune(self, R):  # builder.cpp:141-150
        for u, l in self.lists.items():
            if len(l) > R:
                self.lists[u] = sorted(l, key=lambda e: (np.float32(e[1]), e[0]))[:R]

    def sorted_lists(self):
        return {u: sorted(l, key=lambda e: (np.float32(e[1]), e[0])) for u, l in self.lists.items()}
