"""Sharded build through torch.distributed + NCCL (one rank, one GPU) on the
C5 generator prefix, checked against the single-context build: per-pass
counters and the whole graph.  Run as a script by tests/test_sharded.py (a
process group is per process).  This is the configuration where the
library's stream once raced the NCCL collective (import before the
all-to-all had finished)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(n: int, port: int) -> int:
    import torch
    import torch.distributed as dist
    import datagen
    from paper_2310_20419_b200 import rnnd as R, sharded as SH
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    cfg = datagen.CONFIGS["C5-deep10M"]
    data = datagen.rows(cfg.cfg, cfg.seed, 0, n)
    eng = SH.DeviceShard(data, 0, n)
    p = dict(S=20, R=96, T1=4, T2=15, seed=42)
    st = SH.sharded_build([eng], SH.TorchDistTransport(), n, 1, **p)
    single = R.BuildStats()
    g = R.build(R.VectorStore(data), R.BuildParams(S=20, R=96, T1=4, T2=15, seed=42), single)
    dist.destroy_process_group()
    got = [list(map(int, c)) for c in st.pass_counts]
    want = [[c.removed, c.inserted, c.flag_skips, c.pair_checks] for c in single.pass_counts]
    if got != want:
        print("counters differ")
        return 1
    part, ref = eng.graph(), g.csr
    same = (np.array_equal(part.offsets, ref.offsets) and np.array_equal(part.ids, ref.ids)
            and np.array_equal(part.dists.view(np.uint32), ref.dists.view(np.uint32)))
    print("ok" if same else "graph differs")
    return 0 if same else 1


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]), int(sys.argv[2])))
