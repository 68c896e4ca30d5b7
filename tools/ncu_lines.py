"""Per-source-line warp stall samples from `ncu -i X --page source --csv --print-source cuda,sass` (diagnostic)."""
import csv
import sys

rows = []
fname = None
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] not in ("", "Function Name"):
        try:
            rows.append((int(r[4]), int(r[5]), fname, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in rows)
print("total samples", tot)
lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4]) if len(sys.argv) > 4 else 10**9
sel = [x for x in rows if (len(sys.argv) <= 2 or x[2] == sys.argv[2]) and lo <= x[3] <= hi]
if len(sys.argv) > 3:
    sel.sort(key=lambda x: (x[2], x[3]))
else:
    sel.sort(reverse=True)
    sel = sel[:50]
for s, ni, f, ln, src in sel:
    if s:
        print(f"{100.0 * s / tot:6.2f}% {s:7d} {ni:7d} {f}:{ln:5d}  {src}")
