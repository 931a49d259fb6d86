"""RNN-Descent vs the NN-Descent baseline on the GPU: the comparison of the
reference's acceptance criterion 5 (tests/acceptance.cpp:95-110, :226-235):
a 100k x 128 store with intrinsic dimension 16 (synth_lowdim,
dataset.cpp:145-173, restated here with numpy), RNN-Descent with default
BuildParams against NN-Descent with K = 64, iters = 10.  Prints one JSON line:
device build seconds of both (CUDA events) and their ratio, plus the
graph-quality side (10-NN recall of each graph's lists over 1,000 sampled
vertices, against GPU brute force).

  python tools/compare_nndescent.py [--n 100000]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def splitmix_unit(seed: int, count: int) -> np.ndarray:
    """SplitMix64(seed).unit_float() x count (rng.hpp:19-31)."""
    M = (1 << 64) - 1
    out = np.empty(count, np.float32)
    s = seed
    for i in range(count):
        s = (s + 0x9E3779B97F4A7C15) & M
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z ^= z >> 31
        out[i] = np.float32(z >> 40) * np.float32(1.0 / 16777216.0)
    return out


def mix_seed(seed: int, stream: int) -> int:
    M = (1 << 64) - 1
    st = (seed ^ ((0xD1B54A32D192ED03 * (stream + 1)) & M)) & M
    st = (st + 0x9E3779B97F4A7C15) & M
    z = st
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def synth_lowdim(n: int, d: int, latent: int, seed: int) -> np.ndarray:
    scale = np.float32(1.0 / np.sqrt(np.float32(latent)))
    A = ((splitmix_unit(mix_seed(seed, 0), d * latent) * np.float32(2) - np.float32(1)) * scale)
    A = A.reshape(d, latent)
    Z = splitmix_unit(mix_seed(seed, 1), n * latent).reshape(n, latent)
    return (Z.astype(np.float64) @ A.astype(np.float64).T).astype(np.float32)


def recall10(g, base, R, sample):
    q = R.VectorStore(base[sample])
    gt = R.brute_force_gt(R.VectorStore(base), q, 11)
    hit = tot = 0
    for i, u in enumerate(sample):
        truth = [int(t) for t in np.asarray(gt.ids).reshape(len(sample), 11)[i] if t != u][:10]
        tot += len(truth)
        hit += len(set(truth) & {e.id for e in g.list(int(u))})
    return hit / tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    args = ap.parse_args()
    from paper_2310_20419_b200 import rnnd as R
    base = synth_lowdim(args.n, 128, 16, 44)
    store = R.VectorStore(base)
    dev = R.Device()
    dev.set_data(store)
    R.build(store, R.BuildParams(), device=dev)  # warm-up
    st = R.BuildStats()
    g_rnn = R.build(store, R.BuildParams(), st, device=dev)
    rnn_s = st.seconds
    sample = np.random.default_rng(0).choice(args.n, 1000, replace=False)
    rec_rnn = recall10(g_rnn, base, R, sample)
    ndev = R.Device()
    ndev.set_data(store)
    p = R.NnDescentParams(K=64, iters=10)
    R.build_nndescent(store, p, device=ndev)  # warm-up
    nst = R.BuildStats()
    g_nnd = R.build_nndescent(store, p, nst, device=ndev)
    rec_nnd = recall10(g_nnd, base, R, sample)
    print(json.dumps({
        "workload": f"synth_lowdim {args.n} x 128 (latent 16, seed 44)",
        "rnn_descent": {"params": "S=20 R=96 T1=4 T2=15", "seconds": rnn_s,
                        "recall10_of_lists": rec_rnn, "avg_out_degree": R.degree_stats(g_rnn).avg_out},
        "nn_descent": {"params": "K=64 sample=10 iters=10 pool=128 (deferred join)",
                       "seconds": nst.seconds, "recall10_of_lists": rec_nnd},
        "ratio_rnn_over_nnd": rnn_s / nst.seconds,
        "reference_criterion": "acceptance c5: ratio <= kC5MaxRatio (CPU)",
    }))


if __name__ == "__main__":
    main()
