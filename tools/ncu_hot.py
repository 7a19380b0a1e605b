"""Per-source-line hotspots of one kernel in an .ncu-rep (cuda,sass correlation).

    python tools/ncu_hot.py report.ncu-rep [top]
"""
import csv
import io
import os
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, lines = "?", None, []
    for r in rows:
        if r and r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0]:
            continue
        i_st = hdr.index("Warp Stall Sampling (All Samples)")
        i_in = hdr.index("Instructions Executed")
        st = float(r[i_st] or 0)
        ins = float(r[i_in] or 0)
        lines.append((st, ins, f"{fname}:{r[0]}", r[1].strip()))
    ts = sum(x[0] for x in lines) or 1
    ti = sum(x[1] for x in lines) or 1
    print(f"total stall samples {ts:.0f} total inst {ti:.0f}")
    for st, ins, loc, src in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"stall {st / ts:6.1%}  inst {ins / ti:6.1%}  {loc:22s} | {src[:90]}")


if __name__ == "__main__":
    main()
