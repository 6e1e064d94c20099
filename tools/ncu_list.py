"""Summarises an ncu --csv launch list (gpu__time_duration.sum and, when
captured, dram__bytes_read/write.sum): one row per launch, plus per-kernel
totals.  python tools/ncu_list.py <csv> [--min-ms 0.05]"""
import collections
import csv
import sys

CONV = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "second": 1}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, by = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", "")) * CONV.get(d["Metric Unit"], 1)
            by.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = v
    out = []
    for (i, name), m in by.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        out.append({"id": i, "kernel": name, "ms": t * 1e3, "read_GB": m.get("dram__bytes_read.sum", 0) / 1e9,
                    "write_GB": m.get("dram__bytes_write.sum", 0) / 1e9})
    return out


if __name__ == "__main__":
    mn = float(sys.argv[sys.argv.index("--min-ms") + 1]) if "--min-ms" in sys.argv else 0.05
    L = launches(sys.argv[1])
    for o in L:
        if o["ms"] >= mn:
            gb = (o["read_GB"] + o["write_GB"]) / (o["ms"] / 1e3) if o["ms"] else 0
            print("%4d %-58s %9.3f ms  rd %7.3f  wr %7.3f GB  %6.0f GB/s" % (o["id"], o["kernel"][:58], o["ms"],
                                                                          o["read_GB"], o["write_GB"], gb))
    tot = collections.OrderedDict()
    for o in L:
        k = o["kernel"].split("(")[0][:58]
        t = tot.setdefault(k, [0, 0.0])
        t[0] += 1
        t[1] += o["ms"]
    allms = sum(v[1] for v in tot.values())
    print("\nper kernel: launches, total ms, share")
    for k, (c, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print("%-58s %5d %10.3f %6.1f%%" % (k, c, ms, 100 * ms / allms if allms else 0))
