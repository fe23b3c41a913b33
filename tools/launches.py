"""Summarise an ncu --csv launch list (last N launches): per-kernel metrics."""
import collections
import csv
import sys


def main(path, last=12):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    by = collections.OrderedDict()
    for d in data:
        by.setdefault((d["ID"], d["Kernel Name"].split("(")[0][-40:]), {})[d["Metric Name"]] = d["Metric Value"]
    keys = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__grid_size", "dram__bytes_read.sum"]
    print("id kernel", " ".join(k.split(".")[0].split("__")[-1] for k in keys))
    for (i, k), m in list(by.items())[-last:]:
        print(i, k, " ".join(str(m.get(x, "-")) for x in keys))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
