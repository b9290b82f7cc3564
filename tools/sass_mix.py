"""Instruction mix + stall share per opcode (and per source line with --lines) from
`ncu -i REP --page source --csv --print-source sass` output."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
print(rows[0][1][:100])
h = rows[1]
ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
cnt, stall = collections.Counter(), collections.Counter()
tot = stot = 0
for r in rows[2:]:
    if len(r) <= ie:
        continue
    toks = r[src].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    base = op.split(".")[0] if "--full" not in sys.argv else op
    try:
        n, s = int(r[ie] or 0), int(r[st] or 0)
    except ValueError:
        continue
    cnt[base] += n; stall[base] += s; tot += n; stot += s
print("total warp-inst", tot, "stall samples", stot)
for k, v in cnt.most_common(40):
    print(f"{k:22s} {v:10d} {v / tot:6.3f}  stall {stall[k] / max(stot, 1):6.3f}")
