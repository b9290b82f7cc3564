"""Host-side logic of the multi-GPU sort on CPU: partition ranges and the
exchange protocol over a real 2-process gloo group (sharded.DistExchange)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_13299_b200 import sharded


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_ranges_partition(world):
    rng = np.random.default_rng(world)
    for _ in range(50):
        total, nblocks = int(rng.integers(0, 300000)), int(rng.integers(1, 5000))
        rs = [sharded.shard_ranges(total, nblocks, r, world) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == total and rs[0][2] == 0 and rs[-1][3] == nblocks
        for a, b in zip(rs, rs[1:]):
            assert a[1] == b[0] and a[3] == b[2]
        sizes = [r[1] - r[0] for r in rs]
        assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_banded_block_rows_partition(world):
    """Banded passes: the ranks' block-row ranges partition the pass's block rows
    for every offset dy, and every cell a rank processes lies inside the target
    band it computed for the level (rows [own_lo, own_hi + beta))."""
    for side in (64, 96, 512, 1000, 1024, 4096):
        for beta in (16, 17, 33, 64, 128, 512):
            banded, bands = sharded.level_bands(side, beta, world)
            if not banded:
                assert all(b[2] == 0 and b[3] == side for b in bands)
                continue
            for dy in sorted({0, 1, beta // 2, beta - 1}):
                first_y = dy if dy > 0 else beta
                ranges = [sharded.banded_block_rows(side, beta, dy, world, r) for r in range(world)]
                nby = ranges[0][2]
                assert ranges[0][0] == 0 and ranges[-1][1] == nby
                for a, b in zip(ranges, ranges[1:]):
                    assert a[1] == b[0]
                for r, (lo, hi, _) in enumerate(ranges):
                    if lo == hi:
                        continue
                    y_first = 0 if lo == 0 else first_y + (lo - 1) * beta
                    y_end = min(side, first_y + (hi - 1) * beta)  # end row of block row hi - 1
                    _, _, band_lo, band_hi = bands[r]
                    assert band_lo <= y_first and y_end <= band_hi, (side, beta, dy, world, r)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = sharded.DistExchange()
        n = 64
        res = []
        # PLAS_XCHG_PASS: XPART = 4 doubles per rank (int128 change as two words, count, pad)
        for step, counts in enumerate([(3, 5), (0, 0), (7, 2)]):
            cnt = counts[rank]
            send = torch.zeros(2 * n, dtype=torch.int32)
            for e in range(cnt):
                send[2 * e] = 100 * rank + e          # cell
                send[2 * e + 1] = 1000 * rank + step  # element
            recv = torch.full((2 * n * world,), -1, dtype=torch.int32)
            part = torch.tensor([0.25 * (rank + 1) + step, -1.5 * rank, float(cnt), 0.0], dtype=torch.float64)
            part_all = torch.zeros(4 * world, dtype=torch.float64)
            m = ex(send, recv, part, part_all)
            res.append((m, part_all.tolist(), recv[: 2 * m * world].tolist()))
        # PLAS_XCHG_ALLGATHER: in place inside a byte workspace
        ws = torch.zeros(256, dtype=torch.uint8)
        off, nb = 40, 12
        ws[off + rank * nb: off + (rank + 1) * nb] = torch.arange(nb, dtype=torch.uint8) + 50 * rank
        ex.allgather(ws, off, nb)
        ag = ws[off: off + world * nb].tolist()
        # PLAS_XCHG_ALLTOALL: rank r sends (q + 1) * (r + 2) bytes of value 10 r + q to rank q
        ws2 = torch.zeros(512, dtype=torch.uint8)
        soff, roff = 8, 200
        send_sizes = [(q + 1) * (rank + 2) for q in range(world)]
        recv_sizes = [(rank + 1) * (j + 2) for j in range(world)]
        pos = soff
        for qq in range(world):
            ws2[pos: pos + send_sizes[qq]] = 10 * rank + qq
            pos += send_sizes[qq]
        ex.alltoall(ws2, soff, roff, send_sizes, recv_sizes)
        a2a = ws2[roff: roff + sum(recv_sizes)].tolist()
        q.put((rank, res, ag, a2a))
    finally:
        dist.destroy_process_group()


def test_dist_exchange_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out = {g[0]: g[1] for g in got}
    ags = {g[0]: g[2] for g in got}
    a2as = {g[0]: g[3] for g in got}
    for step, counts in enumerate([(3, 5), (0, 0), (7, 2)]):
        m = max(counts)
        for rank in range(world):
            got_m, part_all, recv = out[rank][step]
            assert got_m == m
            assert part_all == [0.25 * 1 + step, 0.0, float(counts[0]), 0.0,
                                0.25 * 2 + step, -1.5, float(counts[1]), 0.0]
            for r in range(world):
                seg = recv[2 * m * r: 2 * m * (r + 1)]
                for e in range(counts[r]):
                    assert seg[2 * e] == 100 * r + e and seg[2 * e + 1] == 1000 * r + step
        assert out[0][step] == out[1][step]  # identical on every rank
    want = sum(([50 * r + i for i in range(12)] for r in range(world)), [])
    assert ags[0] == want and ags[1] == want
    for rank in range(world):
        exp = []
        for j in range(world):
            exp += [10 * j + rank] * ((rank + 1) * (j + 2))
        assert a2as[rank] == exp
