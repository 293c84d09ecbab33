"""Per-kernel share of device time from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`).
Usage: python profiles/launch_share.py launches.csv [OUT.json]"""
import collections
import csv
import json
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, im, iv, iu = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        try:
            v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        except ValueError:
            continue
        if v != v:  # nan
            continue
        grid = r[hdr.index("Grid Size")] if "Grid Size" in hdr else ""
        name = r[ik].split("(")[0][:60] + " grid" + grid
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    out = [{"kernel": k, "launches": cnt[k], "total_us": round(v, 2), "avg_us": round(v / cnt[k], 3),
            "share": round(v / s, 4)} for k, v in sorted(tot.items(), key=lambda x: -x[1])]
    for d in out:
        print(f"{d['kernel'][:70]:70s} n={d['launches']:4d} avg={d['avg_us']:8.3f}us share={d['share']:.3f}")
    if len(sys.argv) > 2:
        json.dump(out, open(sys.argv[2], "w"), indent=1)


if __name__ == "__main__":
    main()
