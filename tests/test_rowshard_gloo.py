"""Row-sharded application across ranks, host logic on CPU (gloo): the binding rowshard.py ships -- handle exchange,
bind, phase 1 / barrier / phase 2 / barrier, ring order, rank-ordered trace -- must reproduce the single-process
program bit for bit.  The per-rank member is a stand-in for the GPU one with the same contract: its bt lives in a
file-backed shared mapping (the "peer-mapped" memory), its handle is the file's path, its phase 1 stores its rows of bt
into EVERY member's mapping (what transpose_push does over NVLink) and its phase 2 walks the column blocks in ring
order.  On a GPU box the same orchestration drives the C ABI (GpuMember; tests/test_gpu_parity.py)."""
import json
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class MappedMember:
    """Member protocol of rowshard.py on top of oracle/matmul_oracle.c (row-range nests) and shared file mappings."""

    def __init__(self, n, rank, tmp, dtype=0):
        from oracle import cpu
        self.n, self.app, self.tmp = n, cpu.App(n, dtype), Path(tmp)
        self.path = self.tmp / f"bt_rank{rank}.bin"
        self.app.bt = np.memmap(self.path, dtype=self.app.c.dtype, mode="w+", shape=(n, n))
        self.app.bt[:] = np.nan          # poisoned: a block nobody stored shows up
        self.peers, self.rank, self.world = {}, None, None
        self.consumed = []

    def export_handle(self):
        return str(self.path).encode()

    def bind(self, rank, world, handles):
        assert len(handles) == world and handles[rank] == self.export_handle()
        self.rank, self.world = rank, world
        for r, h in enumerate(handles):
            self.peers[r] = self.app.bt if r == rank else np.memmap(h.decode(), dtype=self.app.c.dtype, mode="r+", shape=(self.n, self.n))

    def phase1(self):
        from paper_1806_01430_b200.rowshard import ring_order, row_block
        r0, r1 = row_block(self.n, self.world, self.rank)
        self.app.run_nest(0, r0, r1)       # a[R]
        self.app.run_nest(1, 0, self.n)    # all of b
        self.app.run_nest(2, r0, r1)       # c[R] = 0
        self.app.run_nest(3, r0, r1)       # bt[R] = b[:, R]^T into the own mapping ...
        for dst in ring_order(self.rank, self.world)[1:]:   # ... and into every peer's, ring order
            self.peers[dst][r0:r1] = self.app.bt[r0:r1]
            self.peers[dst].flush()

    def phase2(self):
        from paper_1806_01430_b200.rowshard import ring_order, row_block
        r0, r1 = row_block(self.n, self.world, self.rank)
        self.consumed = ring_order(self.rank, self.world)
        assert not np.isnan(self.app.bt).any(), "a peer's rows of bt have not arrived"
        self.app.run_nest(4, r0, r1)       # c[R] += a[R] . bt^T (the oracle has no column-block form: all blocks at once)
        c = self.app.c
        s = c.dtype.type(0)
        for i in range(r0, r1):
            s = c.dtype.type(s + c[i, i])
        esz = c.dtype.itemsize
        return {"rank": self.rank, "world": self.world, "row0": r0, "rows": r1 - r0, "gpu_ms": 0.0, "exchange_ms": 0.0, "matmul_ms": 0.0,
                "peer_bytes": (r1 - r0) * self.n * esz * (self.world - 1), "partial_trace": float(s)}


def _worker(rank, world, port, n, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    from oracle import cpu
    from paper_1806_01430_b200.rowshard import RowShardedRun, control_group
    dist.init_process_group("gloo", rank=rank, world_size=world)
    member = MappedMember(n, rank, out_dir)
    run = RowShardedRun(member, control_group(120.0))
    res = run.run()
    res = run.run()          # a second individual over the same binding
    ref = cpu.App(n).run()
    r0, r1 = res["rows"]
    ok_c = bool(np.array_equal(member.app.c[r0:r1].view(np.uint64), ref.c[r0:r1].view(np.uint64)))
    ok_bt = bool(np.array_equal(np.asarray(member.app.bt).view(np.uint64), ref.bt.view(np.uint64)))
    Path(out_dir, f"rank{rank}.json").write_text(json.dumps(
        {"rows": [r0, r1], "ok_c": ok_c, "ok_bt": ok_bt, "checksum": res["checksum"], "ref_checksum": ref.checksum,
         "peer_bytes": res["peer_bytes"], "consumed": member.consumed}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,n", [(2, 128), (3, 100)])   # equal 64-aligned blocks; ragged blocks
def test_row_sharded_run_matches_the_single_process_program(tmp_path, world, n):
    mp.spawn(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    outs = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(world)]
    covered = []
    for r, o in enumerate(outs):
        assert o["ok_c"] and o["ok_bt"]
        covered.append(tuple(o["rows"]))
        assert o["peer_bytes"] == 8 * n * (o["rows"][1] - o["rows"][0]) * (world - 1)
        assert o["consumed"] == [(r + d) % world for d in range(world)]     # own block first, then the ring
    assert covered[0][0] == 0 and covered[-1][1] == n
    assert all(covered[i][1] == covered[i + 1][0] for i in range(world - 1))   # a partition of the rows
    assert len({o["checksum"] for o in outs}) == 1
    if n == 128:   # power of two: the trace is exactly 0 whatever the association
        assert outs[0]["checksum"] == outs[0]["ref_checksum"] == 0.0
    else:
        assert abs(outs[0]["checksum"] - outs[0]["ref_checksum"]) < 1e-9


def test_rank_ordered_sum_follows_the_program_dtype():
    sys.path.insert(0, str(ROOT))
    from paper_1806_01430_b200.rowshard import sum_in_rank_order
    parts = [1.0, 2.0 ** -30, -1.0]
    assert sum_in_rank_order(parts, False) == 2.0 ** -30      # double keeps the small term
    assert sum_in_rank_order(parts, True) == 0.0              # float drops it, as the float program's running sum would


def test_row_blocks_partition_and_align():
    sys.path.insert(0, str(ROOT))
    from paper_1806_01430_b200.rowshard import row_block
    for n, world in ((32768, 8), (4096, 4), (4096, 3), (100, 3), (64, 2), (7, 8)):
        blocks = [row_block(n, world, r) for r in range(world)]
        assert blocks[0][0] == 0 and blocks[-1][1] == n
        assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
        if n % 64 == 0 and n // 64 >= world:
            assert all(lo % 64 == 0 and hi % 64 == 0 for lo, hi in blocks)
    assert [row_block(32768, 8, r) for r in (0, 7)] == [(0, 4096), (28672, 32768)]
