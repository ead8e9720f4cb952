"""Per-kernel table from an `ncu --metrics gpu__time_duration.sum --csv` launch
list: launches, total / average duration and share of the profiled range.

    python tools/launch_table.py gpurun_out/step_launches_s8.csv
"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def table(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        if (mi is not None and r[mi] != "gpu__time_duration.sum") or r[ui] not in SCALE:
            continue  # other metrics in the same list (grid size, DRAM bytes)
        us = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        k = r[ki].split("(")[0].replace("void ", "")[:58]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    out = [f"launches {sum(a[0] for a in agg.values())}, total {tot:.1f} us (serialised, cold-cache ncu replay)"]
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:58s} n={n:4d} total={us:10.1f}us avg={us / n:8.2f}us share={us / tot * 100:5.1f}%")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        print(table(p))
