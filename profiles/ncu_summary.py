"""Summarise `ncu --set full` reports (.ncu-rep) into a small JSON + text
table: per launch the duration, DRAM bytes read/written, DRAM/SM/FMA/tensor
utilisation, registers, grid. Usage:
    python profiles/ncu_summary.py OUT.json REP.ncu-rep [REP2 ...]"""
import csv
import io
import json
import subprocess
import sys

BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
METRICS = {
    "duration_us": ("gpu__time_duration.sum", {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}),
    "dram_read_bytes": ("dram__bytes_read.sum", BYTES),
    "dram_write_bytes": ("dram__bytes_write.sum", BYTES),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", None),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", None),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "registers": ("launch__registers_per_thread", None),
    "grid": ("launch__grid_size", None),
    "block": ("launch__block_size", None),
    "smem_per_block": ("launch__shared_mem_per_block", BYTES),
}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:120], "report": rep.split("/")[-1]}
        for key, (m, conv) in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if conv:
                v *= conv.get(units[i], 1)
            d[key] = round(v, 3)
        if "dram_read_bytes" in d:
            d["dram_bytes"] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0)
        res.append(d)
    return res


def main():
    dst, reps = sys.argv[1], sys.argv[2:]
    allk = []
    for rep in reps:
        allk += summarise(rep)
    json.dump(allk, open(dst, "w"), indent=1)
    for d in allk:
        print(f"{d['kernel'][:60]:60s} {d.get('duration_us', 0):9.2f}us dram={d.get('dram_bytes', 0) / 1e6:8.3f}MB "
              f"dram%={d.get('dram_pct', 0):5.1f} fma%={d.get('fma_pipe_pct', 0):5.1f} "
              f"tc%={d.get('tensor_pipe_pct', 0):5.1f} warps%={d.get('warps_active_pct', 0):5.1f}")


if __name__ == "__main__":
    main()
