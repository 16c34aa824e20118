"""Summarise an ncu --set full report (raw page) into CSV: per launch time, DMMA-pipe activity, DRAM
bytes, grid, registers, occupancy, L2 hit rate.  Usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import subprocess
import sys

KEYS = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "time"),
        ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_active_pct"),
        ("dram__bytes_read.sum", "dram_read"), ("dram__bytes_write.sum", "dram_write"),
        ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
        ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct")]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    cols = [(hdr.index(k), name) for k, name in KEYS if k in hdr]
    w = csv.writer(sys.stdout)
    w.writerow([name + (f" ({units[i]})" if units[i] else "") for i, name in cols])
    for r in rows[2:]:
        w.writerow([r[i].split("(")[0].strip() if name == "kernel" else r[i] for i, name in cols])


if __name__ == "__main__":
    main(sys.argv[1])
