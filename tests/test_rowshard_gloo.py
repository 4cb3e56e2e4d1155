"""Row-sharded application across ranks, host logic on CPU (gloo): the partition, the all-gather of bt
(equal blocks -> in-place all_gather_into_tensor; ragged blocks -> per-owner broadcast) and the rank-ordered
trace must reproduce the single-process program bit for bit.  The per-rank compute is a numpy engine backed
by the oracle's row-range nests; on a GPU box the same orchestration drives the C ABI (GpuEngine)."""
import json
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleEngine:
    """Engine protocol of rowshard.py on top of oracle/matmul_oracle.c (row-range nests)."""

    def __init__(self, n, dtype=0):
        from oracle import cpu
        self.n, self.app = n, cpu.App(n, dtype)
        self._bt = torch.from_numpy(self.app.bt)   # shares memory with the numpy array

    def fill_rows(self, gene, r0, r1):
        self.app.run_nest({0: 0, 2: 1, 4: 2}[gene], r0, r1)

    def transpose_rows(self, r0, r1):
        self.app.run_nest(3, r0, r1)

    def matmul_rows(self, r0, r1):
        self.app.run_nest(4, r0, r1)

    def trace_rows(self, r0, r1):
        c = self.app.c
        s = c.dtype.type(0)
        for i in range(r0, r1):
            s = c.dtype.type(s + c[i, i])
        return float(s)

    def bt_tensor(self):
        return self._bt

    def sync(self):
        pass


def _worker(rank, world, port, n, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    from oracle import cpu
    from paper_1806_01430_b200.rowshard import run_row_sharded
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = OracleEngine(n)
    res = run_row_sharded(eng)
    ref = cpu.App(n).run()
    r0, r1 = res["rows"]
    ok_c = bool(np.array_equal(eng.app.c[r0:r1].view(np.uint64), ref.c[r0:r1].view(np.uint64)))
    ok_bt = bool(np.array_equal(eng.app.bt.view(np.uint64), ref.bt.view(np.uint64)))
    Path(out_dir, f"rank{rank}.json").write_text(json.dumps(
        {"rows": [r0, r1], "ok_c": ok_c, "ok_bt": ok_bt, "checksum": res["checksum"], "ref_checksum": ref.checksum,
         "gathered_bytes": res["gathered_bytes"]}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,n", [(2, 128), (3, 100)])   # equal 64-aligned blocks; ragged blocks
def test_row_sharded_run_matches_the_single_process_program(tmp_path, world, n):
    mp.spawn(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    outs = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(world)]
    covered = []
    for o in outs:
        assert o["ok_c"] and o["ok_bt"]
        covered.append(tuple(o["rows"]))
        assert o["gathered_bytes"] == 8 * n * (n - (o["rows"][1] - o["rows"][0]))
    assert covered[0][0] == 0 and covered[-1][1] == n
    assert all(covered[i][1] == covered[i + 1][0] for i in range(world - 1))   # a partition of the rows
    assert len({o["checksum"] for o in outs}) == 1
    if n == 128:   # power of two: the trace is exactly 0 whatever the association
        assert outs[0]["checksum"] == outs[0]["ref_checksum"] == 0.0
    else:
        assert abs(outs[0]["checksum"] - outs[0]["ref_checksum"]) < 1e-9


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
