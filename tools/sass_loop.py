"""Opcode histogram and listing of the hottest loop of one kernel in an ncu report
(source page, SASS): python tools/sass_loop.py rep.ncu-rep [launch_index] > out.txt"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
i = [k for k, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[i]
data = [r for r in rows[i + 1:] if len(r) == len(h) and r[h.index("Instructions Executed")].isdigit()]
ie, src = h.index("Instructions Executed"), h.index("Source")
cnt = collections.Counter(int(r[ie]) for r in data if int(r[ie]) > 0)
top = max(cnt, key=lambda n: n * cnt[n])
seq = [r[src].strip() for r in data if int(r[ie]) == top]
ops = collections.Counter()
for s in seq:
    op = s.split()[0] if not s.startswith("@") else s.split()[1]
    ops[op.split(".")[0]] += 1
print("loop count", top, "instructions", len(seq))
print(ops.most_common(40))
print("\n".join(seq))
