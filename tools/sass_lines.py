"""Per-source-line instruction counts: join `ncu --page source --print-source sass --csv`
output (SASS addresses + Instructions Executed) with `nvdisasm -gi` line info of the
same cubin.  python tools/sass_lines.py NCU_SASS.csv ALL.sass MANGLED_KERNEL [top]"""
import collections, csv, re, sys
ncu_csv, sass, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
loc_of = {}
inside = False
cur = None
for line in open(sass):
    if line.startswith(".text."):
        inside = line.strip().rstrip(":") == ".text." + kern
        continue
    if not inside:
        continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', line)
    if m:
        if cur is None:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]+)\*/", line)
    if m:
        if cur is not None:
            loc_of[int(m.group(1), 16)] = cur
            last = cur
        else:
            loc_of[int(m.group(1), 16)] = last if loc_of else ("?", 0)
        cur = None
rows = list(csv.reader(open(ncu_csv)))
h = rows[1]
ia, ie, st = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) > ie]
base = int(data[0][ia], 16)
cnt, stall = collections.Counter(), collections.Counter()
tot = stot = 0
for r in data:
    off = int(r[ia], 16) - base
    loc = loc_of.get(off, ("?", 0))
    n, s = int(r[ie] or 0), int(r[st] or 0)
    cnt[loc] += n; stall[loc] += s; tot += n; stot += s
print("total", tot, "mapped offsets", len(loc_of))
for loc, v in cnt.most_common(top):
    print(f"{loc[0]}:{loc[1]:<5d} {v:10d} {v / tot:6.3f}  stall {stall[loc] / max(stot, 1):6.3f}")
