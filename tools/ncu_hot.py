"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[1:]:
    if len(r) <= iss:
        continue
    try:
        data.append((int(r[iss]), r[ia], r[isrc].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", len(data))
for s, a, src in sorted(data, reverse=True)[:top]:
    print("%6d %5.1f%%  %s  %s" % (s, 100.0 * s / tot, a[-5:], src))
# aggregate by opcode
agg = {}
for s, a, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    agg[op] = agg.get(op, 0) + s
print("by opcode:", sorted(agg.items(), key=lambda x: -x[1])[:12])
