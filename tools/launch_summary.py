"""Per-kernel totals of an ncu --csv gpu__time_duration launch list (run here)."""
import collections
import csv
import sys


def main(path, width=90):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[h.index("Metric Value")].replace(",", ""))
        unit = r[h.index("Metric Unit")]
        v = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        k = r[h.index("Kernel Name")][:width]
        tot[k][0] += 1
        tot[k][1] += v
    s = sum(v[1] for v in tot.values())
    print(f"total {s:.1f} us in {sum(v[0] for v in tot.values())} launches")
    for k, v in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"{v[0]:5d} {v[1]:9.1f} us {v[1] / v[0]:8.2f} us/launch {100 * v[1] / s:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
