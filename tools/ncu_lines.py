"""Attribute ncu SASS-level stall samples / instructions to CUDA source lines.

    python tools/ncu_lines.py <ncu sass csv> <cubin> <mangled kernel name> [top]

The ncu csv is `ncu -i rep --page source --csv --print-source sass`; the cubin is
extracted from the built object (`cuobjdump -xelf all build_obj/ops_p4.o`).  Rows
are joined by instruction order within the function (nvdisasm -g line info)."""
import collections
import csv
import os
import re
import subprocess
import sys


def main(csv_path, cubin, fn, top=40):
    rows = list(csv.reader(open(csv_path)))[1:]
    h, R = rows[0], rows[1:]
    iS, iI = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    sass = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
    start = next(i for i, l in enumerate(sass) if l.startswith(".text." + fn + ":"))
    cur, lines = None, []
    for l in sass[start + 1:]:
        if l.startswith(".text.") or "\t.section" in l:
            break
        m = re.search(r'//## File "(.*)", line (\d+)', l)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l):
            lines.append(cur)
    n = min(len(lines), len(R))
    iW, iX = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Excessive")
    samp, inst, wf, wx = (collections.Counter() for _ in range(4))

    def num(x):
        return float(x.replace(",", "")) if x not in ("", "-") else 0.0

    for k in range(n):
        samp[lines[k]] += int(R[k][iS])
        inst[lines[k]] += int(R[k][iI])
        wf[lines[k]] += num(R[k][iW])
        wx[lines[k]] += num(R[k][iX])
    tot = sum(samp.values())
    print(f"instructions matched {n} of {len(R)} (sass {len(lines)}); samples {tot}; "
          f"shared wavefronts {sum(wf.values()):.0f} (excessive {sum(wx.values()):.0f})")
    key = wf if os.environ.get("BY_WAVEFRONTS") else samp
    for loc, _ in key.most_common(top):
        print(f"{100 * samp[loc] / tot:5.1f}%  inst {inst[loc]:10d}  smem wf {wf[loc]:10.0f} exc {wx[loc]:9.0f}  {loc}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
