"""Histogram of executed SASS opcodes from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
si, ei, sa = h.index("Source"), h.index("Instructions Executed"), h.index("# Samples")
agg, samp = collections.Counter(), collections.Counter()
tot = 0
for r in rows[hi + 1:]:
    if len(r) <= ei:
        continue
    op = r[si].split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    n = int(r[ei].replace(",", "") or 0)
    agg[o] += n
    samp[o] += int(r[sa].replace(",", "") or 0)
    tot += n
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print("total warp-instr %d  per-unit %.3f" % (tot, tot / norm))
for o, n in agg.most_common(40):
    print("%-22s %12d  %6.2f%%  per-unit %.3f  samples %d" % (o, n, 100.0 * n / tot, n / norm, samp[o]))
