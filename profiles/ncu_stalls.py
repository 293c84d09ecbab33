"""Warp-stall sample shares per kernel from an ncu --set full report (pc sampling):
python profiles/ncu_stalls.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    pre = "smsp__pcsamp_warps_issue_stalled_"
    for r in rows[2:]:
        st = {}
        for i, x in enumerate(h):
            if x.startswith(pre) and not x.endswith("_not_issued"):
                try:
                    st[x[len(pre):]] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        print(f"{r[h.index('Kernel Name')][:70]}  ({int(tot)} samples)")
        for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]:
            print(f"   {k:<28} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main()
