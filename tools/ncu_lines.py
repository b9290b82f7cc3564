"""Aggregate an ncu source-page (SASS) export by CUDA source line.

usage: python tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_SUBSTRING [launch_index]

Exports the SASS page of the first matching launch, disassembles the same
kernel from the .so with line info (nvdisasm -gi), maps instruction offsets to
file:line and prints stall samples and executed instructions per line.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_page(report, kernel, launch):
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kernel}", "--launch-skip", str(launch), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    name = rows[0][1]
    hdr = rows[1]
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break  # next launch / kernel block
        if len(r) == len(hdr) and r[0] != "Address":
            data.append(dict(zip(hdr, r)))
    return name, data


def line_map(lib, mangled_hint):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cubin)], capture_output=True,
                         text=True).stdout
    funcs = {}
    cur = None
    chain = []
    fresh = True
    for line in txt.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", line)
        if m:
            cur = m.group(1)
            funcs[cur] = {}
            chain = []
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            if fresh:
                chain = []
                fresh = False
            chain.append((os.path.basename(m.group(1)), int(m.group(2))))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
        if m and cur is not None:
            # innermost frame, and the innermost frame outside common.cuh
            inner = chain[0] if chain else ("?", 0)
            own = next((c for c in chain if c[0] != "common.cuh"), inner)
            funcs[cur][int(m.group(1), 16)] = (inner, own)
            fresh = True
    cands = [f for f in funcs if all(h in f for h in mangled_hint)]
    cands.sort(key=len)
    return funcs, cands


def main():
    report, lib, kernel = sys.argv[1:4]
    launch = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    name, data = sass_page(report, kernel, launch)
    print("kernel:", name)
    hints = sys.argv[5].split(",") if len(sys.argv) > 5 else [kernel]
    funcs, cands = line_map(lib, hints)
    if not cands:
        print("no function matches", hints, list(funcs)[:20])
        return
    fmap = funcs[cands[0]]
    base = int(data[0]["Address"], 16)
    agg = collections.defaultdict(lambda: [0, 0, 0])
    tot_s = 0
    level = 1 if os.environ.get("NCU_LINES_OWN") else 0
    for d in data:
        off = int(d["Address"], 16) - base
        loc = fmap.get(off, (("?", 0), ("?", 0)))[level]
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        e = int(d["Instructions Executed"] or 0)
        agg[loc][0] += s
        agg[loc][1] += e
        agg[loc][2] += 1
        tot_s += s
    tot_e = sum(v[1] for v in agg.values())
    print(f"function {cands[0]}  samples {tot_s}  warp-instructions {tot_e}")
    limit = int(os.environ.get("NCU_LINES_TOP", "40"))
    for loc, (s, e, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:limit]:
        print(f"{100 * s / max(tot_s, 1):5.1f}% samples {100 * e / max(tot_e, 1):5.1f}% instr  {n:4d} sass  {loc[0]}:{loc[1]}")


if __name__ == "__main__":
    main()
