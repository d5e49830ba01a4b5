"""The N>1 path is independent replicas (the single-GPU solve path
does not shard; bench.py --gpus N runs one replica per rank and reports the
max-over-ranks time).  World-size-2 gloo test on CPU: both ranks build the
same decomposition bit for bit, and the max-over-ranks reduction used by
bench.py behaves as specified."""
import os

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch

    from paper_1909_08734_b200 import api, inputs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = api.Problem("sphere", h=0.1, p=3, workers=2)
    P.decompose(inputs.rcb_partition(P.active_cp, 8), 2, "oras", 4.0, 40.0)
    h = np.uint64(1469598103934665603)
    for j in range(P.n_sub):
        L = P.local(j)
        for a in (L["ptr"], L["col"], L["val"]):
            h = np.uint64((int(h) * 1099511628211 + int(np.frombuffer(a.tobytes(), np.uint8).sum())) % (1 << 64))
    t = torch.tensor([float(int(h) % (1 << 52))], dtype=torch.float64)
    allh = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allh, t)
    tm = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    out[rank] = (float(allh[0]), float(allh[1]), float(tm))
    dist.destroy_process_group()


def test_two_replicas_identical_and_max_over_ranks():
    port = 29500 + (os.getpid() % 1000)
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0][0] == res[0][1] == res[1][0] == res[1][1]
    assert res[0][2] == res[1][2] == 2.0
