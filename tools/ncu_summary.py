#!/usr/bin/env python
"""Boil an .ncu-rep (ncu --set full) down to the handful of per-launch numbers the roofline
discussion uses; writes CSV to stdout.  Run here (no GPU needed): ncu only parses the report."""
import csv
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static", "launch__grid_size", "launch__block_size",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "derived__lts__lts2xbar_bytes.sum.per_second", "l1tex__m_xbar2l1tex_read_bytes.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
]


def traffic(rep, n, out_path):
    """Merge `kernel@N -> dram bytes per launch` of this report into a JSON table (bench.py reads it)."""
    import json
    import re
    from pathlib import Path
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    ir, iw, ik, it = (hdr.index(k) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "Kernel Name", "gpu__time_duration.sum"))
    acc = {}
    for r in rows[2:]:
        m = re.search(r"(\w+_kernel)", r[ik])
        name = (m.group(1) if m else r[ik])[: -len("_kernel")] if m else r[ik]
        b = float(r[ir]) * scale[units[ir]] + float(r[iw]) * scale[units[iw]]
        dur_us = float(r[it]) * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(units[it], 1.0)
        if any(k in name for k in ("ozaki", "dmma", "3xtf32", "split_planes")) and dur_us < 20.0:
            continue   # a guarded launch that did nothing (auto mode: the other path took the product): not the kernel's traffic
        acc.setdefault(name, []).append((b, float(r[it])))
    p = Path(out_path)
    table = json.loads(p.read_text()) if p.exists() else {}
    for name, vals in acc.items():
        table[f"{name}@{n}"] = {"bytes_per_launch": sum(v[0] for v in vals) / len(vals), "launches": len(vals),
                                "ncu_duration_" + units[it]: sum(v[1] for v in vals) / len(vals), "report": Path(rep).name}
    p.write_text(json.dumps(table, indent=1, sort_keys=True) + "\n")


def main():
    if sys.argv[1] == "--traffic":   # --traffic <rep> <N> <out.json>
        return traffic(sys.argv[2], int(sys.argv[3]), sys.argv[4])
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    cols = [hdr.index("Kernel Name")] + [hdr.index(k) for k in KEEP if k in hdr]
    w = csv.writer(sys.stdout)
    w.writerow([hdr[c] + (f" [{units[c]}]" if units[c] else "") for c in cols])
    for r in rows[2:]:
        w.writerow([r[c] for c in cols])


if __name__ == "__main__":
    main()
