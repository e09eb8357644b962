"""Summarise ncu reports: duration, DRAM traffic/throughput, issue, pipes, stalls.
    python tools/ncu_summary.py report.ncu-rep [...]"""
import csv
import io
import subprocess
import sys


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
]


def main():
    for path in sys.argv[1:]:
        hdr, units, rows = raw(path)
        for r in rows:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            print(f"== {path}: {d.get('Kernel Name', '')[:60]}")
            for k, nm in KEYS:
                if k in d:
                    print(f"   {nm:12s} {d[k]} {u[k]}")
            pipes = {k.split("pipe_")[1].split(".")[0]: float(d[k]) for k in hdr
                     if k.startswith("sm__inst_executed_pipe_") and
                     k.endswith(".avg.pct_of_peak_sustained_active") and d[k]}
            print("   pipes%      ", {p: round(v, 1) for p, v in pipes.items() if v > 3})
            st = {k.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", ""): float(d[k]) for k in hdr
                if k.startswith("smsp__average_warps_issue_stalled_") and
                k.endswith("_per_issue_active.ratio") and d[k]}
            print("   stalls      ", {p: round(v, 2) for p, v in sorted(st.items(),
                                                                     key=lambda x: -x[1])
                                     if v > 0.2})


if __name__ == "__main__":
    main()
