"""Regenerates the inputs of tests/golden/builds.json cases (test helper)."""
import numpy as np


def data_for(case):
    from oracle import oracle as O
    if case["kind"] == "uniform":
        return O.synth_uniform(case["n"], case["d"], case["data_seed"])
    if case["kind"] == "grid":  # heavy exact ties and duplicate points
        u = O.synth_uniform(case["n"], case["d"], case["data_seed"])
        return (np.round(u * 8.0) / 8.0).astype(np.float32)
    import datagen
    return datagen.rows(case["cfg"], case["data_seed"], 0, case["n"])
