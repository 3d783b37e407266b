#!/usr/bin/env python
"""Attribute an ncu source-page SASS CSV (--page source --csv --print-source sass) to source
lines with their full inline chain (nvdisasm -gi of the kernel's object file): where the
warp-stall samples and executed instructions of one kernel go, by innermost source line.

  python scripts/sass_lines.py SASS.csv OBJ.o MANGLED_KERNEL_NAME [top]
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_map(obj, name):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    start = sass.index(f".text.{name}:")
    end = sass.find(".section", start + 10)
    m, group = {}, []
    for ln in sass[start:end if end > 0 else None].split("\n"):
        f = re.search(r'//## File "[^"]*/([^"/]+)", line (\d+)(.*)', ln)
        if f:
            chain = [f"{f.group(1)}:{f.group(2)}"] + [f"{a}:{b}" for a, b in
                                                      re.findall(r'inlined at "[^"]*/([^"/]+)", line (\d+)', f.group(3))]
            group.append(chain)
            continue
        a = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if a:
            if group:
                cur = max(group, key=len)  # the innermost location carries the longest chain
                group = []
            m[int(a.group(1), 16)] = cur if "cur" in dir() else ["?"]
    return m


def main():
    path, obj, name = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    base = int(data[0][0], 16)
    lm = line_map(obj, name)

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (ValueError, KeyError):
            return 0.0

    samp, inst, stl = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for r in data:
        ch = lm.get(int(r[0], 16) - base, ["?"])
        key = " <- ".join(ch[:3])
        samp[key] += f(r, "Warp Stall Sampling (All Samples)")
        inst[key] += f(r, "Instructions Executed")
        for s in stalls:
            stl[key][s[6:]] += f(r, s)
    T = sum(samp.values())
    for key, v in samp.most_common(top):
        print(f"{100 * v / T:5.1f}%  inst {inst[key]:12.0f}  {key[:90]:90s} {stl[key].most_common(2)}")


if __name__ == "__main__":
    main()
