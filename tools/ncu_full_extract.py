"""Extract the judged raw metrics of an `ncu --set full` report into a small JSON
(profiles/): per launch the duration, DRAM bytes, throughputs, occupancy, issue,
and the top stall reasons.  usage: python tools/ncu_full_extract.py REP OUT.json "source text" """
import csv, io, json, subprocess, sys
rep, out, source = sys.argv[1], sys.argv[2], sys.argv[3]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic"]
res = {"source": source, "launches": []}
for v in rows[2:]:
    d = {"kernel": v[h.index("Kernel Name")]}
    for w in want:
        if w in h:
            d[w] = f"{v[h.index(w)]} {units[h.index(w)]}".strip()
    st = []
    for i, w in enumerate(h):
        if w.startswith("smsp__average_warps_issue_stalled_") and w.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), w[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    d["top_stalls_per_issue"] = {k: round(x, 3) for x, k in sorted(st, reverse=True)[:6]}
    res["launches"].append(d)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
