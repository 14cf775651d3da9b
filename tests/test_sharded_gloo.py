"""world_size-2 gloo test of the mode-1-sharded STR schedule: the test-side
re-statement of libstr's sharded step (tests/_sharded_schedule.py; three sum-allreduces per
batch at sites C1, C2, C2') equals the unsharded fp64 oracle after init and every batch."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, k, nb, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests._sharded_schedule import ShardedSTR
        from oracle.stream import StreamingTR
        from workloads import make_stream
        from workloads.gen import paper_view
        s = make_stream(name)
        cfg = s.cfg
        w = cfg.dims[0] // world

        def shard(x):
            return np.ascontiguousarray(x[..., rank * w:(rank + 1) * w]).astype(np.float64)

        Xi = s.init_slab()
        st = ShardedSTR(s.init_cores(), shard(Xi), k, world, rank)
        orc = StreamingTR(paper_view(Xi), s.init_cores()) if rank == 0 else None
        errs = []
        for b in range(nb):
            Xb = s.batch(b)
            st.update(shard(Xb))
            cores = [st.core(n) for n in range(1, cfg.N + 1)]
            if rank == 0:
                orc.update(paper_view(Xb))
                errs.append(max(np.linalg.norm(c - o) / np.linalg.norm(o) for c, o in zip(cores, orc.cores)))
        if rank == 0:
            q.put(errs)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,k", [("T5", 2), ("T4", 1), ("T3", 1)])
def test_sharded_schedule_matches_oracle(name, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, k, 2, q)) for r in range(2)]
    for p in procs:
        p.start()
    errs = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert max(errs) < 1e-10, errs
