"""Summarise an ncu launch list (development): per-kernel totals and shares
plus the per-launch table, in the format of profiles/r1_launches_*.txt.

usage: python tests/dev_launch_summary.py <ncu --csv log> "<command it profiled>"
(the log of `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --clock-control none -c N --csv --log-file ...`)."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    head = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[head]
    ii, ik, im, iu, iv = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                                "Metric Value"))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3,
             "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "KB": 1e-6, "MB": 1e-3,
             "GB": 1.0}
    launches = OrderedDict()
    for r in rows[head + 1:]:
        d = launches.setdefault(int(r[ii]), {"name": r[ik]})
        v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        d[r[im]] = v
    return launches


def short(name):
    name = name.replace("(int)", "").replace("(bool)", "")
    return name.split("(")[0] if "<" not in name else name[: name.index(">") + 1]


def main():
    path, cmd = sys.argv[1], sys.argv[2]
    L = load(path)
    tot = sum(d.get("gpu__time_duration.sum", 0.0) for d in L.values())
    per = OrderedDict()
    for d in L.values():
        k = short(d["name"])
        p = per.setdefault(k, [0, 0.0, 0.0])
        p[0] += 1
        p[1] += d.get("gpu__time_duration.sum", 0.0)
        p[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    print("# ncu launch list of '%s', first %d launches" % (cmd, len(L)))
    print("# per-launch times are cold-cache and serialised (ncu --metrics, --clock-control none)")
    print("\n## per kernel")
    for k, (n, t, b) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print("%-60s n=%4d time=%9.3f ms share=%6.3f avg=%9.1f us dram/launch=%7.3f GB"
              % (k, n, t / 1e3, t / tot, t / n, b / n))
    print("\n## launches (id, kernel, time us, dram read GB, dram write GB)")
    for i, d in L.items():
        print("%5d %-72s %9.1f %8.3f %8.3f" % (i, short(d["name"])[:72], d.get("gpu__time_duration.sum", 0),
                                              d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)))


if __name__ == "__main__":
    main()
