"""Per-opcode instruction / stall-sample / shared-wavefront breakdown of an ncu report."""
import collections
import csv
import subprocess
import sys


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    si, st, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    wf, wfi = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
    by, cnt, wfs, wfsi = (collections.Counter() for _ in range(4))
    tot = 0
    for r in rows[2:]:
        try:
            s, n = float(r[st] or 0), float(r[ie] or 0)
        except ValueError:
            continue
        toks = r[si].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        by[op] += s
        cnt[op] += n
        tot += s
        try:
            wfs[op] += float(r[wf] or 0)
            wfsi[op] += float(r[wfi] or 0)
        except ValueError:
            pass
    for op, s in by.most_common(22):
        print(f"{op:10s} samples {s / tot * 100:5.1f}%  inst {cnt[op]:12.0f}  smem_wf {wfs[op]:10.0f} ideal {wfsi[op]:10.0f}")
    print("total inst", sum(cnt.values()))


if __name__ == "__main__":
    main(sys.argv[1])
