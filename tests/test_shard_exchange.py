"""Index sharding on CPU with torch.distributed/gloo, world sizes 2 and 4.

Each rank builds its level-h send buffer from the library's layout (bf_shard_pairs, the same index
functions the kernels use), runs the all-to-all over gloo exactly as the plan does over NCCL (G equal
contiguous blocks), and checks the received pairs against the library's receive layout and against
the ownership rule written out here from its definition: before the exchange pair (a, b) at level h
lives on the rank given by b's top g bits, after it on the rank given by a's top g bits.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_04128_b200 import bf

CASES = [(12, 4), (16, 5), (22, 6)]


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
        g = world.bit_length() - 1
        for LN, l0 in CASES:
            h = LN // 2
            N = 1 << LN
            send = bf.shard_pairs(LN, l0, world, rank, 0)
            recv_expect = bf.shard_pairs(LN, l0, world, rank, 1)
            second = bf.shard_pairs(LN, l0, world, rank, 2)
            # ownership from the definition: p = a 2^h + b (LN - h = h)
            a_s, b_s = send >> h, send & ((1 << h) - 1)
            assert np.all(b_s >> (h - g) == rank), "send side owns the pairs whose b has top bits = rank"
            assert len(np.unique(send)) == N // world
            # the send buffer is destination-major: block d holds exactly the pairs whose a has top bits d
            blk = N // world // world
            for d in range(world):
                assert np.all(a_s[d * blk:(d + 1) * blk] >> (h - g) == d)
            # second-half order: the contiguous global range of this rank's x-rows
            assert np.array_equal(second, np.arange(rank * N // world, (rank + 1) * N // world))
            # the exchange, as bf_apply performs it (equal contiguous blocks)
            out = torch.empty(N // world, dtype=torch.int64)
            dist.all_to_all_single(out, torch.from_numpy(send))
            got = out.numpy()
            assert np.array_equal(got, recv_expect), "received layout == the kernels' receive layout"
            a_r = got >> h
            assert np.all(a_r >> (h - g) == rank), "after the exchange a rank holds the pairs of its x-rows"
            assert np.array_equal(np.sort(got), second)
            # the same exchange moving whole coefficient blocks (r rows x nv vectors per pair, as the level-h
            # launch writes them in send order), checked word for word against the receive layout the
            # second-half kernel reads (bfs::recv_index, exported as bf_shard_pairs(which = 1))
            if LN <= 16:
                R, nv = 4, 3
                t = np.arange(R)[:, None]
                v = np.arange(nv)[None, :]
                blocks = (send[:, None, None] << 16) | (t << 8) | v          # content names (pair, row, vector)
                out = torch.empty(blocks.size, dtype=torch.int64)
                dist.all_to_all_single(out, torch.from_numpy(np.ascontiguousarray(blocks).ravel()))
                recv = out.numpy().reshape(-1, R, nv)
                expect = (recv_expect[:, None, None] << 16) | (t << 8) | v
                assert np.array_equal(recv, expect), "received blocks == receive layout, word for word"
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 4])
def test_index_shard_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_shard_validation():
    with pytest.raises(bf.BFError):
        bf.shard_pairs(12, 4, 3, 0, 0)       # not a power of two
    with pytest.raises(bf.BFError):
        bf.shard_pairs(8, 4, 4, 0, 0)        # h - g < 2
    with pytest.raises(bf.BFError):
        bf.shard_pairs(12, 4, 2, 2, 0)       # rank out of range
