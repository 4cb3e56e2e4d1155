"""Row-sharded run of the matrix application across the GPUs of one box -- the torchrun binding
of the fused path in the C ABI (`mmx_shard_export / bind / phase1 / phase2`, include/mmx.h, csrc/executor.cu).

For very large N one individual is spread over G ranks (one process per GPU):

    rank g owns rows R_g = [r0, r1) of a, c and bt          (contiguous blocks, 64-row aligned when possible)
    init-a, zero-c       : rows R_g only                     (index-generated: no communication)
    init-b               : the whole of b, locally            (index-generated; cheaper than exchanging it)
    transpose + exchange : ONE kernel.  bt[R_g][:] = b[:][R_g]^T is stored into the bt of EVERY member through
                           peer-mapped pointers (NVLink stores): the transpose is the all-gather.  No collective
                           library, no staging buffer.  E*N^2*(G-1)/G bytes leave each GPU.
    matmul               : c[R_g][:] += a[R_g][:] . bt^T, walked column block by column block in ring order
                           starting with the member's own rows of bt; block s waits (on the device) only for member
                           s's "stored everywhere" event, so the math on blocks that have arrived overlaps the
                           transfers still in flight
    trace                : partial sum over the diagonal entries in R_g, then a rank-ordered sum on the host

What crosses the process boundary through torch.distributed is CONTROL only: the 128-byte handles of each member's bt
and ready event (once, `all_gather_object`), two host barriers per run (every ready event is recorded before a peer
enqueues its wait; nobody overwrites a bt a peer is still reading), and the 8-byte partial traces.  Use a gloo group
for it (`control_group()`): the data path never touches NCCL.

`Member` is what the orchestration needs from a rank.  `GpuMember` drives the C ABI; the CPU (gloo) tests plug in a
member whose "peer-mapped bt" is a file-backed shared mapping, so the handle exchange, the ring order, the barriers
and the rank-ordered trace are exercised across real processes without a GPU.
"""
from __future__ import annotations

import time
from typing import Protocol

import torch.distributed as dist


def row_block(n: int, world: int, rank: int, align: int = 64) -> tuple[int, int]:
    """Contiguous, nearly equal row blocks; boundaries are multiples of `align` when n allows it (the tiled
    transpose and the GEMM tiles then never straddle a block edge).  Same rule as shard_block in executor.cu."""
    unit = align if n % align == 0 and n // align >= world else 1
    units = n // unit
    lo = (units * rank) // world * unit
    hi = (units * (rank + 1)) // world * unit
    return lo, hi


def ring_order(rank: int, world: int) -> list[int]:
    """Owners of the column blocks in the order member `rank` consumes them (its own first): at any instant the
    members read -- and, in the exchange kernel, write -- different peers."""
    return [(rank + d) % world for d in range(world)]


class Member(Protocol):
    """One rank's share of the row-sharded individual (mirrors mmx_shard_* one to one)."""

    n: int

    def export_handle(self) -> bytes: ...                                  # mmx_shard_export
    def bind(self, rank: int, world: int, handles: list[bytes]) -> None: ...  # mmx_shard_bind
    def phase1(self) -> None: ...   # fills + fused transpose/exchange; records the member's ready event
    def phase2(self) -> dict: ...   # ring-ordered column blocks gated by the owners' events, partial trace; waits


class GpuMember:
    """The member on this rank's GPU: a capi.Context with one slot (include/mmx.h)."""

    def __init__(self, ctx, slot: int = 0):
        self.ctx, self.slot, self.n = ctx, slot, ctx.n

    def export_handle(self) -> bytes:
        return self.ctx.shard_export(self.slot)

    def bind(self, rank, world, handles):
        self.ctx.shard_bind(rank, world, handles, self.slot)

    def phase1(self):
        self.ctx.shard_phase1(self.slot)

    def phase2(self):
        return self.ctx.shard_phase2(self.slot)


def control_group(timeout_s: float = 600.0):
    """A gloo group over all ranks for handles, barriers and the 8-byte partial traces (host-side control only)."""
    import datetime
    return dist.new_group(backend="gloo", timeout=datetime.timedelta(seconds=timeout_s))


class RowShardedRun:
    """Binds a member into the group once (handle exchange), then runs individuals.

    Every rank constructs it with its own member and calls run() the same number of times."""

    def __init__(self, member: Member, group=None, dtype_is_f32: bool = False):
        self.member, self.group, self.f32 = member, group, dtype_is_f32
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        mine = member.export_handle()
        if self.world > 1:
            table: list = [None] * self.world
            dist.all_gather_object(table, mine, group=group)
        else:
            table = [mine]
        member.bind(self.rank, self.world, table)
        self._barrier()   # every member is bound (its peers' mappings are open) before anyone stores into a peer

    def _barrier(self):
        if self.world > 1:
            dist.barrier(group=self.group)

    def run(self) -> dict:
        """One pass of the application.  Every rank returns the same checksum; `rows` is this rank's block of c."""
        t0 = time.perf_counter()
        self.member.phase1()
        self._barrier()          # every ready event is recorded before anyone enqueues a wait on it
        st = self.member.phase2()
        self._barrier()          # nobody starts the next run's stores while a peer still reads this run's bt
        wall = time.perf_counter() - t0
        partial = float(st["partial_trace"])
        if self.world > 1:
            parts: list = [None] * self.world
            dist.all_gather_object(parts, partial, group=self.group)
        else:
            parts = [partial]
        checksum = sum_in_rank_order(parts, self.f32)
        return {"checksum": checksum, "rows": (st["row0"], st["row0"] + st["rows"]), "rank": self.rank, "world": self.world,
                "peer_bytes": int(st["peer_bytes"]), "gpu_ms": st["gpu_ms"], "exchange_ms": st["exchange_ms"],
                "matmul_ms": st["matmul_ms"], "wall_s": wall}


def sum_in_rank_order(parts, f32: bool) -> float:
    """Block by block in rank order, in the program's dtype: the association the program's own running sum would use
    across the blocks (mmx_shard_run_local does the same in-process)."""
    if f32:
        import numpy as np
        s = np.float32(0.0)
        for p in parts:
            s = np.float32(s + np.float32(p))
        return float(s)
    s = 0.0
    for p in parts:
        s += float(p)
    return s


def run_row_sharded(member: Member, group=None, dtype_is_f32: bool = False) -> dict:
    """Bind + one run (convenience for tests)."""
    return RowShardedRun(member, group, dtype_is_f32).run()
