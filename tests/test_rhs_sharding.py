"""RHS sharding (BASELINE config 4 "RHS are sharded across 1/2/4/8 GPUs") on CPU with
torch.distributed/gloo: bench.py's rank q applies columns [q nrhs/G, (q+1) nrhs/G) of the ONE seeded
batch.  Each rank generates only its columns; gathered in rank order they are the full batch, bitwise,
and every column belongs to exactly one rank (strong scaling: the ranks together apply the batch once).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from paper_1803_04128_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n, nrhs, seed = 1 << 10, 12, 3
        c0, c1 = bench.rhs_columns(nrhs, world, rank)
        mine = W.rhs(n, nrhs, seed, cols=range(c0, c1))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([c1 - c0]))
        cap = max(int(s) for s in sizes)
        buf = torch.zeros((cap, n, 2), dtype=torch.float32)
        buf[: c1 - c0] = torch.from_numpy(np.ascontiguousarray(mine.T).view(np.float32).reshape(c1 - c0, n, 2))
        got = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(got, buf)
        cols = [g[: int(s)].numpy() for g, s in zip(got, sizes)]
        full = np.concatenate(cols, axis=0).view(np.complex64).reshape(-1, n).T
        assert np.array_equal(full, W.rhs(n, nrhs, seed)), "rank blocks concatenate to the batch"
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 4])
def test_rhs_partition_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


@pytest.mark.parametrize("nrhs,world", [(256, 1), (256, 2), (256, 8), (8, 8), (13, 4), (3, 4)])
def test_rhs_columns_cover_once(nrhs, world):
    spans = [bench.rhs_columns(nrhs, world, q) for q in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == nrhs
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
