"""Hot loop of an ncu source-page CSV (ncu -i rep --page source --csv): instruction count,
opcode histogram and listing with stall samples: python tools/src_loop.py file.source.csv [-l]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[i]
ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[i + 1:] if len(r) > ie and r[ie].isdigit() and int(r[ie]) > 0]
cnt = collections.Counter(int(r[ie]) for r in data)
top = max(cnt, key=lambda n: n * cnt[n])
seq = [r for r in data if int(r[ie]) == top]
ops = collections.Counter()
for r in seq:
    s = r[src].split()
    ops[(s[1] if s[0].startswith("@") else s[0]).split(".")[0]] += 1
print(rows[0][1][:90])
print("total", sum(int(r[ie]) for r in data), "loop count", top, "instructions", len(seq))
print(ops.most_common(40))
if "-l" in sys.argv:
    for r in seq:
        print(r[st].rjust(6), r[src][:100])
