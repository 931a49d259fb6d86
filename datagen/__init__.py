"""Seeded synthetic inputs for the BASELINE.json configs (datagen/datagen.cpp).

Test and bench infrastructure (libdatagen.so), not part of the product
library.  Row i depends only on (config, seed, i); queries are the held-out
rows n .. n+nq-1 of the same stream.  Host-side generation (no GPU needed).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdatagen.so")
_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `make -C datagen`")
        L = C.CDLL(LIB_PATH)
        L.dg_synth_dim.restype = C.c_uint32
        L.dg_synth_dim.argtypes = [C.c_int]
        L.dg_synth.restype = C.c_int
        L.dg_synth.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                               C.POINTER(C.c_float)]
        _LIB = L
    return _LIB


@dataclass(frozen=True)
class Config:
    name: str
    cfg: int
    n: int
    nq: int
    seed: int

    @property
    def d(self) -> int:
        return int(lib().dg_synth_dim(self.cfg))


# BASELINE.json configs[0..4]; seeds: C1 0 and C5 1 are given, C2-C4 chosen
C1 = Config("C1-gmm128-20k", 1, 20_000, 1_000, 0)
C2 = Config("C2-siftlike-1M", 2, 1_000_000, 10_000, 2)
C3 = Config("C3-gistlike-1M", 3, 1_000_000, 1_000, 3)
C4 = Config("C4-deeplike-1M", 4, 1_000_000, 10_000, 4)
C5 = Config("C5-deep10M", 5, 10_000_000, 10_000, 1)
CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}


def rows(cfg: int, seed: int, row0: int, nrows: int) -> np.ndarray:
    L = lib()
    d = int(L.dg_synth_dim(cfg))
    out = np.empty((nrows, d), np.float32)
    rc = L.dg_synth(cfg, seed, row0, nrows, out.ctypes.data_as(C.POINTER(C.c_float)))
    if rc != 0:
        raise ValueError(f"dg_synth failed (cfg={cfg})")
    return out


def base(c: Config, n: int | None = None) -> np.ndarray:
    return rows(c.cfg, c.seed, 0, c.n if n is None else n)


def queries(c: Config, nq: int | None = None, n: int | None = None) -> np.ndarray:
    return rows(c.cfg, c.seed, c.n if n is None else n, c.nq if nq is None else nq)
