"""Multi-GPU mode is replicas only: each rank solves its
own system, the only collective is the max-over-ranks of the timing.  This
exercises bench.py's replica bookkeeping with world_size 2 over gloo on CPU."""
import os
import socket
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    t = 1.0 + rank  # rank 1 is the slow replica
    mx = bench.replica_max(t, ws, "cpu")
    out[rank] = (bench.replica_seed(42, rank), mx, bench.whole_job_seconds_per_system(mx, 5, ws))
    dist.barrier()
    dist.destroy_process_group()


def test_replicas_over_gloo_world_size_2():
    ws, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
        res = dict(out)
    assert res[0][0] != res[1][0]                         # distinct systems per replica
    assert res[0][1] == res[1][1] == 2.0                  # max over ranks, identical on every rank
    assert abs(res[0][2] - 2.0 / (5 * 2)) < 1e-15        # whole-job seconds per system
