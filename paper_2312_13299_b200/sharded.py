"""Multi-GPU PLAS sort: one grid sharded across the ranks of a process group.

Design.  Every rank keeps a full replica of the sort
state and runs the same level/pass loop.  Each pass's groups -- which are
disjoint by construction (plas.py:118-121, 196-223) -- are split into
contiguous, balanced per-rank ranges; a rank reassigns only its own groups,
then the ranks all-gather
  * their fp64 partial distance changes and moved-cell counts (16 B each), and
  * their moved cells as (cell, element) int32 pairs (~3.6 % of their cells),
every rank applies the others' moves (the moved element's f32 row comes from
its own element-order copy of the features, so rows never travel) and runs
the identical controller on the partials summed in rank order.  Draws are
identical on every rank (NumPy-exact host draws in PARITY mode, counter-based
Philox in DEVICE mode), so all replicas stay bit-identical.  The level blur and
level statistics are computed redundantly per rank in this version.

The exchange runs through torch.distributed (NCCL over NVLink on one box); the
library calls back into Python at the exchange point of each pass.
``EmulatedGroup`` runs the same protocol for `world` ranks as threads on one
device (tests: no kernel ever waits on another rank's kernel, the host
rendezvous orders them).
"""

import threading
from dataclasses import dataclass

import numpy as np


@dataclass
class ShardSpec:
    rank: int
    world: int
    exchange: object  # callable(send, recv, part, part_all) -> m


def shard_ranges(total_groups, nblocks, rank, world):
    """This rank's [g_lo, g_hi) groups and [b_lo, b_hi) blocks of a pass
    (host mirror of common.cuh set_pass_geometry_base)."""
    return (total_groups * rank // world, total_groups * (rank + 1) // world,
            nblocks * rank // world, nblocks * (rank + 1) // world)


class DistExchange:
    """The exchange step over a torch.distributed process group (NCCL on GPUs)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        # the collective is chosen once, from the backend: NCCL has the fused
        # all_gather_into_tensor; other backends (gloo in the CPU tests) take
        # the list form.  Runtime errors propagate (a retry on a broken
        # communicator could leave the ranks in different collectives).
        self.fused = str(dist.get_backend(group)).lower() == "nccl"

    def _all_gather(self, out, inp):
        if self.fused:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
        else:
            self.dist.all_gather(list(out.chunk(self.world)), inp, group=self.group)

    def __call__(self, send, recv, part, part_all):
        self._all_gather(part_all, part)
        m = int(part_all.view(self.world, 2)[:, 1].max().item())
        if m > 0:
            self._all_gather(recv[: 2 * m * self.world], send[: 2 * m].contiguous())
        return m


class EmulatedGroup:
    """`world` ranks as host threads on one device: the all-gathers are copies."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def exchange(self, rank):
        def ex(send, recv, part, part_all):
            import torch
            torch.cuda.synchronize()
            self.slots[rank] = (send, part)
            self.barrier.wait()
            part_all.copy_(torch.cat([self.slots[r][1] for r in range(self.world)]))
            m = int(part_all.view(self.world, 2)[:, 1].max().item())
            for r in range(self.world):
                recv[2 * m * r: 2 * m * (r + 1)].copy_(self.slots[r][0][: 2 * m])
            torch.cuda.synchronize()
            self.barrier.wait()  # every rank has read the slots before the next pass refills them
            return m
        return ex


def sort_on_device_sharded(features, config, rank, world, exchange, initial_perm=None):
    """One rank's share of a sharded sort: CUDA tensor in, (CUDA int64 perm, report) out.
    Every rank must call it with the same features and config."""
    import torch
    from . import _lib
    from .plas import SortPlan, _validate
    t, n, side = _validate(features)
    _lib.lib()
    if not isinstance(t, torch.Tensor):
        t = torch.from_numpy(np.ascontiguousarray(t))
    t = t.to("cuda").contiguous()
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    ip = None
    if initial_perm is not None:
        ip = _lib.to_device(np.asarray(initial_perm, dtype=np.int64), torch.int64)
    rep = SortPlan(n, t.shape[1], config).run(t, perm, ip, None, ShardSpec(rank, world, exchange))
    return perm, rep


def sort_grid_sharded(features, config=None, group=None):
    """sort_grid (plas.py:289-296) on every rank of a torch.distributed group;
    returns the int64 host permutation (identical on all ranks)."""
    import torch.distributed as dist
    from .plas import SortConfig
    ex = DistExchange(group)
    perm, _ = sort_on_device_sharded(features, config or SortConfig(), dist.get_rank(group),
                                     dist.get_world_size(group), ex)
    return perm.cpu().numpy()


def sort_emulated(features, config, world, initial_perm=None):
    """Run a `world`-rank sharded sort as threads on the current device; returns
    the per-rank (perm numpy, report) list."""
    grp = EmulatedGroup(world)
    out = [None] * world
    errs = []

    def run(r):
        try:
            p, rep = sort_on_device_sharded(features, config, r, world, grp.exchange(r), initial_perm)
            out[r] = (p.cpu().numpy(), rep)
        except Exception as exc:  # surfaced below
            errs.append(exc)
            grp.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errs:
        raise errs[0]
    return out
