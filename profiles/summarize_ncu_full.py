"""Key columns of an `ncu --page raw --csv` export (one row per kernel):
duration, DRAM bytes and throughput, tensor-pipe and SM utilisation, L2 hit
rate, grid and registers.  Usage: python summarize_ncu_full.py raw.csv > summary.csv"""
import csv
import sys

COLS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_pct"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
        ("lts__t_sector_hit_rate.pct", "l2_hit_pct"), ("launch__grid_size", "grid"),
        ("launch__registers_per_thread", "regs")]


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = rows[0]
    units = rows[1]
    w = csv.writer(sys.stdout)
    w.writerow(["kernel"] + [f"{n} ({units[hdr.index(c)]})" if c in hdr else n for c, n in COLS])
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        w.writerow([d.get("Kernel Name", "?").split("(")[0]] + [d.get(c, "") for c, _ in COLS])


if __name__ == "__main__":
    main(sys.argv[1])
