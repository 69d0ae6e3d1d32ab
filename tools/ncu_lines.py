"""Instructions executed and stall samples per CUDA source line of the first kernel in an ncu
report (--page source, cuda,sass view): python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if r and r[0] == "Line No")
iE, iS = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
fn0 = next(r[1] for r in rows if r and r[0] == "Function Name")
recs = []
fname, func = "", ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Function Name":
        func = r[1]
    elif r[0].isdigit() and func == fn0:
        num = lambda x: int(x) if x.strip().isdigit() else 0  # noqa: E731
        recs.append((num(r[iE]), num(r[iS]), fname, int(r[0]), r[1].strip()))
tot = sum(x[0] for x in recs)
tst = sum(x[1] for x in recs)
print(f"{fn0[:80]}\ntotal instructions {tot}, stall samples {tst}")
for e, s, f, ln, src in sorted(recs, reverse=True)[:top]:
    print(f"{f[:14]:14s}:{ln:5d} {100 * e / tot:5.1f}% inst {100 * s / max(1, tst):5.1f}% stall  {src[:80]}")
