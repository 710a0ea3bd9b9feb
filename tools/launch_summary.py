"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel count,
total and mean time, optionally only the last `--last` launches of each kernel."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((d["Kernel Name"], d["Grid Size"], float(d["Metric Value"]) / 1e3))
    return out


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return name.split("(")[0][:70]


if __name__ == "__main__":
    launches = load(sys.argv[1])
    agg = collections.OrderedDict()
    for k, g, us in launches:
        a = agg.setdefault(short(k), [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%-72s %6d  %10.1f us  %8.2f us/launch  %5.1f%%" % (k, c, us, us / c, 100 * us / tot))
    print("total %.1f ms" % (tot / 1e3))
