"""Multi-GPU PLAS sort: one grid sharded across the ranks of a process group.

Design.  Every rank keeps a replica of the grid
(features and element indices) and runs the same level/pass loop:

* banded levels (beta * world <= side): rank r owns rows
  [Y_r, Y_r+1), Y_r = side r / world, and each pass it takes the block rows
  that start there -- row bands aligned to the pass's block tiling, which
  move with the pass offset dy.  It computes the level's target only on the
  rows its blocks can reach, [Y_r, Y_r+1 + beta): the direct and tile blur
  tiers read the halo rows from the replica, the FFT tier splits its axis-0
  transforms by columns and swaps band pieces with one all-to-all;
* replicated levels (the top levels, beta * world > side): each pass's groups
  are split into even contiguous ranges and every rank blurs the whole grid.

After each pass the ranks all-gather their exact 128-bit distance changes and
moved-cell counts (32 B each) and their moved cells as (cell, element) int32
pairs (~3.6 % of their cells); every rank applies the others' moves (the
moved element's f32 row comes from its own element-order copy of the
features, so rows never travel) and runs the identical controller.  The level
start distance sum is exchanged the same way (128-bit partials of each rank's
own rows).  Fixed-point partials add exactly, so the sort is bit-identical to
one GPU for any world size.  Draws are identical on every rank (NumPy-exact
host draws in PARITY mode, counter-based Philox in DEVICE mode).

The exchange runs through torch.distributed (NCCL over NVLink on one box); the
library calls back into Python at the exchange points (plas_sort_args.exchange,
include/plas_b200.h).  ``EmulatedGroup`` runs the same protocol for `world`
ranks as threads on one device (tests: no kernel ever waits on another rank's
kernel, the host rendezvous orders them).
"""

import threading
from dataclasses import dataclass

import numpy as np


@dataclass
class ShardSpec:
    rank: int
    world: int
    exchange: object  # callable(send, recv, part, part_all) -> m


def level_bands(side, beta, world):
    """Per rank (own_lo, own_hi, band_lo, band_hi) rows of a level and whether it
    is banded (host mirror of plas_sort's level set-up): banded when
    beta * world <= side; own rows [side r / world, side (r+1) / world); the
    target band adds the beta rows a block can reach below them.  Replicated
    levels keep the whole grid as band."""
    banded = beta * world <= side
    out = []
    for r in range(world):
        lo, hi = side * r // world, side * (r + 1) // world
        out.append((lo, hi, lo if banded else 0, min(side, hi + beta) if banded else side))
    return banded, out


def banded_block_rows(side, beta, dy, world, rank):
    """This rank's [by_lo, by_hi) block rows of a banded pass with offset dy
    (host mirror of common.cuh set_pass_geometry_base): the block rows whose
    first row y0(by) (0 for by = 0, first_y + (by - 1) beta after) lies in the
    rank's own rows."""
    first_y = dy if dy > 0 else beta
    nby = 1 + (side - first_y + beta - 1) // beta if first_y < side else 1

    def first_by(Y):
        if Y <= 0:
            return 0
        by = 1 if Y <= first_y else 1 + (Y - first_y + beta - 1) // beta
        return min(by, nby)

    own_lo, own_hi = side * rank // world, side * (rank + 1) // world
    return first_by(own_lo), (nby if own_hi >= side else first_by(own_hi)), nby


def shard_ranges(total_groups, nblocks, rank, world):
    """This rank's [g_lo, g_hi) groups and [b_lo, b_hi) blocks of a pass
    (host mirror of common.cuh set_pass_geometry_base)."""
    return (total_groups * rank // world, total_groups * (rank + 1) // world,
            nblocks * rank // world, nblocks * (rank + 1) // world)


class DistExchange:
    """The exchange steps over a torch.distributed process group (NCCL on GPUs)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
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
        """PLAS_XCHG_PASS: partials (XPART doubles per rank), then the moved cells."""
        from ._lib import XPART
        self._all_gather(part_all, part)
        m = int(part_all.view(self.world, XPART)[:, 2].max().item())
        if m > 0:
            self._all_gather(recv[: 2 * m * self.world], send[: 2 * m].contiguous())
        return m

    def allgather(self, ws, off, nbytes):
        """PLAS_XCHG_ALLGATHER: in place, rank r's piece at ws[off + r nbytes]."""
        view = ws[off: off + self.world * nbytes]
        mine = view[self.rank * nbytes: (self.rank + 1) * nbytes].clone()
        self._all_gather(view, mine)

    def alltoall(self, ws, send_off, recv_off, send_sizes, recv_sizes):
        """PLAS_XCHG_ALLTOALL: byte segments in rank order at ws[send_off], ws[recv_off]."""
        send = ws[send_off: send_off + sum(send_sizes)]
        recv = ws[recv_off: recv_off + sum(recv_sizes)]
        self.dist.all_to_all_single(recv, send, output_split_sizes=list(recv_sizes),
                                    input_split_sizes=list(send_sizes), group=self.group)


class _EmulatedRank:
    """One rank's exchange endpoints of an EmulatedGroup (copies between the ranks' buffers)."""

    def __init__(self, grp, rank):
        self.grp = grp
        self.rank = rank
        self.world = grp.world

    def _rendezvous(self, item):
        import torch
        torch.cuda.synchronize()
        self.grp.slots[self.rank] = item
        self.grp.barrier.wait()

    def _done(self):
        import torch
        torch.cuda.synchronize()
        self.grp.barrier.wait()  # every rank has read the slots before they are refilled

    def __call__(self, send, recv, part, part_all):
        import torch
        from ._lib import XPART
        self._rendezvous((send, part))
        slots = self.grp.slots
        part_all.copy_(torch.cat([slots[r][1] for r in range(self.world)]))
        m = int(part_all.view(self.world, XPART)[:, 2].max().item())
        for r in range(self.world):
            recv[2 * m * r: 2 * m * (r + 1)].copy_(slots[r][0][: 2 * m])
        self._done()
        return m

    def allgather(self, ws, off, nbytes):
        self._rendezvous(ws)
        for r in range(self.world):
            if r != self.rank:
                ws[off + r * nbytes: off + (r + 1) * nbytes].copy_(
                    self.grp.slots[r][off + r * nbytes: off + (r + 1) * nbytes])
        self._done()

    def alltoall(self, ws, send_off, recv_off, send_sizes, recv_sizes):
        self._rendezvous((ws, send_off, list(send_sizes)))
        pos = recv_off
        for j in range(self.world):
            wsj, soff, ssz = self.grp.slots[j]
            src = soff + sum(ssz[: self.rank])
            assert ssz[self.rank] == recv_sizes[j]
            ws[pos: pos + recv_sizes[j]].copy_(wsj[src: src + recv_sizes[j]])
            pos += recv_sizes[j]
        self._done()


class EmulatedGroup:
    """`world` ranks as host threads on one device: the collectives are copies."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def exchange(self, rank):
        return _EmulatedRank(self, rank)


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
