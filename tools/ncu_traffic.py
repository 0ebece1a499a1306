"""Turn an `ncu --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum` log of tools/prof_variant.py into profiles/ncu_traffic_*.json
(the launches of K.p, mass and f_int are grouped by kernel name, in order of
first appearance: with the z-slab schedule K.p and mass are 64 launches each,
f_int 8).  Run here, no GPU."""
import csv
import json
import sys
from collections import defaultdict


def main(log, out):
    rows = [r for r in csv.reader(open(log)) if len(r) > 10]
    hdr = rows[0]
    iid, iname, imet, iunit, ival = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                                             "Metric Value"))
    launches = defaultdict(dict)
    names = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "ms": 1.0,
             "msecond": 1.0}
    for r in rows[1:]:
        k = int(r[iid])
        names[k] = r[iname]
        launches[k][r[imet]] = float(r[ival].replace(",", "")) * scale[r[iunit]]
    ids = sorted(launches)
    res = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     "--clock-control none --cache-control none (steady state), tools/prof_variant.py (config 2: K.p, mass, f_int; launches grouped by "
                     "kernel name); tools/ncu_traffic.py",
           "kernel_kp": names[ids[0]]}
    order = []
    for k in ids:
        if names[k] not in order:
            order.append(names[k])
    for j, op in enumerate(("kp", "mass", "fint")):
        sel = [k for k in ids if names[k] == order[j]]
        res["kernel_" + op] = order[j]
        rd = sum(launches[k]["dram__bytes_read.sum"] for k in sel)
        wr = sum(launches[k]["dram__bytes_write.sum"] for k in sel)
        res[op] = {"launches": len(sel), "time_ms_sum": sum(launches[k]["gpu__time_duration.sum"] for k in sel),
                   "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
