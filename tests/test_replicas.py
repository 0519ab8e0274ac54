"""Multi-rank path of the bench on CPU (gloo, world_size 2): replicas-only
aggregation = max time over ranks, summed updates."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, upd = (10.0, 100) if rank == 0 else (25.0, 300)
    t, u = bench.reduce_replicas(ms, upd, torch.device("cpu"), world)
    out[rank] = (t, u)
    dist.destroy_process_group()


def test_replica_aggregation_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert out[r] == (25.0, 400.0)
