"""Instruction mix and stall samples per SASS opcode from `ncu --page source --csv` output."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ops, stall, tot = collections.Counter(), collections.Counter(), 0
for r in rows[2:]:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    n = int(r[ie])
    t = r[src].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    op = op.split(".")[0]
    ops[op] += n
    tot += n
    stall[op] += int(r[st] or 0)
print("total warp instructions", tot)
for op, n in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print("%-10s %12d %5.1f%%  stall samples %d" % (op, n, 100 * n / tot, stall[op]))
