"""Row-sharded run of the matrix application across the GPUs of one box.

For very large N one individual is spread over G ranks (one process per GPU):

    rank g owns rows R_g = [r0, r1) of a, c and bt          (contiguous blocks, 64-row aligned when possible)
    init-a, zero-c       : rows R_g only                     (index-generated: no communication)
    init-b               : the whole of b, locally            (index-generated; cheaper than exchanging it)
    transpose            : bt[R_g][:] = b[:][R_g]^T           (rows R_g of bt = columns R_g of b)
    ALL-GATHER bt        : the one exchange step of the path  (E*N^2*(G-1)/G bytes received per GPU)
    matmul               : c[R_g][:] += a[R_g][:] . bt^T      (needs all of bt)
    trace                : partial sum over the diagonal entries in R_g, then a rank-ordered sum

The collective runs through torch.distributed on a tensor that ALIASES the library's own device array
(`mmx_device_ptr`), so no staging copy is made: NCCL writes straight into the bt that the matmul kernel
reads.  The engine interface below is what the orchestration needs from a rank; `GpuEngine` drives the C ABI,
and the CPU (gloo) tests plug in a numpy engine to check the partition / gather / reduction logic bit for bit.
"""
from __future__ import annotations

from typing import Protocol

import numpy as np
import torch
import torch.distributed as dist


def row_block(n: int, world: int, rank: int, align: int = 64) -> tuple[int, int]:
    """Contiguous, nearly equal row blocks; boundaries are multiples of `align` when n allows it (the tiled
    transpose and the GEMM tiles then never straddle a block edge)."""
    unit = align if n % align == 0 and n // align >= world else 1
    units = n // unit
    lo = (units * rank) // world * unit
    hi = (units * (rank + 1)) // world * unit
    return lo, hi


class Engine(Protocol):
    n: int

    def fill_rows(self, gene: int, r0: int, r1: int) -> None: ...      # genes 0, 2, 4
    def transpose_rows(self, r0: int, r1: int) -> None: ...             # gene 6
    def matmul_rows(self, r0: int, r1: int) -> None: ...                # gene 8
    def trace_rows(self, r0: int, r1: int) -> float: ...                # gene 11
    def bt_tensor(self) -> torch.Tensor: ...                            # (n, n) view of bt for the collective
    def sync(self) -> None: ...


class _CudaAlias:
    """Minimal __cuda_array_interface__ carrier so torch can alias a raw device pointer."""

    def __init__(self, ptr: int, n: int, np_dtype):
        self.__cuda_array_interface__ = {
            "shape": (n, n), "typestr": np.dtype(np_dtype).str, "data": (ptr, False), "version": 3, "strides": None,
        }


class GpuEngine:
    def __init__(self, ctx, device: int = 0):
        from . import capi
        self.ctx, self.n, self.capi = ctx, ctx.n, capi
        alias = _CudaAlias(ctx.device_ptr(capi.ARRAY_BT), ctx.n, ctx.np_dtype)
        self._bt = torch.as_tensor(alias, device=torch.device("cuda", device))

    def fill_rows(self, gene, r0, r1):
        self.ctx.run_loop_rows(gene, r0, r1 - r0)

    def transpose_rows(self, r0, r1):
        self.ctx.run_loop_rows(6, r0, r1 - r0)

    def matmul_rows(self, r0, r1):
        self.ctx.run_loop_rows(8, r0, r1 - r0)

    def trace_rows(self, r0, r1):
        return self.ctx.run_loop_rows(11, r0, r1 - r0)

    def bt_tensor(self):
        return self._bt

    def sync(self):
        torch.cuda.synchronize()


def run_row_sharded(engine: Engine, group=None) -> dict:
    """One pass of the application with rows sharded over the ranks of `group`.  Every rank returns the same
    checksum; `rows` says which block of c this rank holds."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = engine.n
    r0, r1 = row_block(n, world, rank)

    engine.fill_rows(0, r0, r1)        # a[R_g]
    engine.fill_rows(2, 0, n)          # all of b (local, index-generated)
    engine.fill_rows(4, r0, r1)        # c[R_g] = 0
    engine.transpose_rows(r0, r1)      # bt[R_g] = b[:, R_g]^T
    engine.sync()

    gathered_bytes = 0
    if world > 1:
        bt = engine.bt_tensor()
        blocks = [row_block(n, world, r) for r in range(world)]
        if len({hi - lo for lo, hi in blocks}) == 1:
            # equal blocks: in-place all-gather (this rank's input is its own slice of the output)
            dist.all_gather_into_tensor(bt, bt[r0:r1], group=group)
        else:
            for src, (lo, hi) in enumerate(blocks):   # ragged blocks: one broadcast per owner
                if hi > lo:
                    dist.broadcast(bt[lo:hi], src=dist.get_global_rank(group, src) if group is not None else src, group=group)
        gathered_bytes = bt.element_size() * n * (n - (r1 - r0))
        engine.sync()

    engine.matmul_rows(r0, r1)
    partial = engine.trace_rows(r0, r1)

    if world > 1:
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dev = engine.bt_tensor().device
        mine = torch.tensor([partial], dtype=torch.float64, device=dev)
        parts = [p.to(dev) for p in parts]
        dist.all_gather(parts, mine, group=group)
        checksum = 0.0
        for p in parts:                # rank order: the same association on every rank
            checksum += float(p.item())
    else:
        checksum = partial
    return {"checksum": checksum, "rows": (r0, r1), "rank": rank, "world": world, "gathered_bytes": gathered_bytes}
