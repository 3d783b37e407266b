"""List the local-memory spill instructions (STL/LDL) of one round-loop kernel with their
inline chain (nvdisasm -gi), to see which of them sit inside hot loops.
  python scripts/spills.py OBJ.o [pol bidir fuse stats]"""
import os
import re
import subprocess
import sys
import tempfile

obj = sys.argv[1]
pol, bidir, fuse, stats = (sys.argv[2:6] + ["0", "0", "0", "0"])[:4] if len(sys.argv) > 2 else ("0", "0", "0", "0")
name = f"_ZN4sssp15sssp_round_loopILi{pol}ELb{stats}ELb{fuse}ELb{bidir}EEEvNS_9RunParamsE"
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
start = sass.index(f".text.{name}:")
end = sass.find(".section", start + 10)
body = sass[start:end if end > 0 else None].split("\n")
cur = ""
for line in body:
    m = re.search(r'//## File "[^"]*/([^"/]+)", line (\d+)(.*)', line)
    if m:
        chain = [f"{m.group(1)}:{m.group(2)}"] + [f"{a}:{b}" for a, b in re.findall(r'inlined at "[^"]*/([^"/]+)", line (\d+)', m.group(3))]
        cur = " <- ".join(chain)
        continue
    if re.search(r"\b(STL|LDL)", line):
        a = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        print(f"{a.group(1)}  {a.group(2)[:40]:40s}  {cur}")
