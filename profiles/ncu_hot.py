"""Summarise an `ncu --page source --csv --print-source sass` dump: the
instructions with the most warp-stall samples (first kernel in the file)."""
import csv
import sys


def main(path, n=30):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "Address":
            if hdr is not None:
                break  # only the first kernel
            hdr = r
            continue
        if hdr is not None and len(r) == len(hdr):
            data.append(r)
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    i_ex = hdr.index("Instructions Executed")
    f = lambda x: float(x) if x not in ("", None) else 0.0
    tot = sum(f(r[i_s]) for r in data)
    print(f"total stall samples {tot:.0f}, {len(data)} instructions")
    for r in sorted(data, key=lambda r: -f(r[i_s]))[:n]:
        print(f"{r[0]:>6} {f(r[i_s]) / tot * 100:5.1f}% ex={r[i_ex]:>8}  {r[i_src][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
