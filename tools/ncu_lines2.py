"""Per-CUDA-source-line instruction counts and stall samples of one kernel from
`ncu -i REP --page source --csv --print-source cuda,sass` (the cuda rows carry
the per-line totals).  usage: python tools/ncu_lines2.py REP.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
out, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        try:
            ie = int(r[7] or 0)
            st = int(r[4] or 0)
        except ValueError:
            continue
        if ie or st:
            out.append((ie, st, fname, r[0], r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
stot = sum(o[1] for o in out) or 1
print("total warp-inst", tot, "stall samples", stot)
for ie, st, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{ie / tot:6.3f} {st / stot:6.3f} {f}:{ln:5s} {src}")
