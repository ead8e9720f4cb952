"""Summarise .ncu-rep files: per-kernel duration, DRAM bytes / throughput,
tensor-pipe activity, occupancy (reads `ncu -i ... --page raw --csv`)."""
import csv
import io
import subprocess
import sys

WANT = [
    ("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "dram_rd_MB"), ("dram__bytes_write.sum", "dram_wr_MB"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_%"),
    ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h = rows[0]
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, short in WANT:
            if k in h:
                i = h.index(k)
                v = r[i]
                u = units[i]
                if short in ("dram_rd_MB", "dram_wr_MB"):
                    f = float(v.replace(",", ""))
                    f = f / 1e6 if u == "byte" else f * (1e3 if u == "Gbyte" else 1) if u in ("Mbyte", "Gbyte") else f / 1e3 if u == "Kbyte" else f
                    v = f"{f:.2f}"
                if short == "us":
                    f = float(v.replace(",", ""))
                    f = f / 1e3 if u == "nsecond" else f * 1e3 if u == "msecond" else f
                    v = f"{f:.2f}"
                if short == "kernel":
                    v = v.split("(")[0][-48:]
                d[short] = v
        res.append(d)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        for d in summarize(p):
            print("  " + " | ".join(f"{k}={v}" for k, v in d.items()))
