"""Summarise an `ncu -i X.ncu-rep --page raw --csv` dump: one block per launch
with time, DRAM bytes, cache hit rates, occupancy, IPC and the warp-stall
breakdown from PC sampling.

    python tools/ncu_raw_summary.py gpurun_out/prof2/flat_full_raw.csv [title]
"""
import csv
import io
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__maximum_warps_per_active_cycle_pct", "theoretical occupancy %"),
    ("smsp__inst_executed.sum", "instructions executed"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM, active)"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.find('"ID"'):])))
    hdr, units = rows[0], rows[1]
    print(title)
    for r in rows[2:]:
        print()
        print(" " + r[hdr.index("Kernel Name")][:110])
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {label:<34} {r[i]:>18} {units[i]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith(STALL) and not h.endswith("_not_issued"):
                try:
                    st.append((float(r[i].replace(",", "")), h[len(STALL):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st)
        if tot > 0:
            print("  warp stall reasons (pc sampling):")
            for v, name in sorted(st, reverse=True)[:8]:
                print(f"    {name:<28} {100 * v / tot:5.1f} %")


if __name__ == "__main__":
    main()
