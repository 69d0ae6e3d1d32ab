"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# one kernel (first) only
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
iS, iN, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
data = []
for r in rows[1:]:
    if len(r) != len(h) or not r[iS].isdigit():
        break
    data.append((int(r[iS]), r[iN].strip(), int(r[iE] or 0)))
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", len(data))
for s, src, ex in sorted(data, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}%  exec={ex:8d}  {src}")
# opcode histogram by executed count
from collections import Counter
c = Counter()
cs = Counter()
for s, src, ex in data:
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    c[op.split(".")[0]] += ex
    cs[op.split(".")[0]] += s
print("executed by opcode:", c.most_common(15))
print("stall samples by opcode:", cs.most_common(15))
