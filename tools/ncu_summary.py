"""Summarise one kernel of an ncu --set full report into a small JSON (profiles/).
    python tools/ncu_summary.py rep.ncu-rep "kernel description" [algorithmic_bytes]"""
import csv, io, json, subprocess, sys

rep, desc = sys.argv[1], sys.argv[2]
alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
m = {}
for w in want:
    if w in hdr:
        i = hdr.index(w)
        try:
            m[w] = {"value": float(vals[i].replace(",", "")), "unit": units[i]}
        except ValueError:
            m[w] = {"value": vals[i], "unit": units[i]}
out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?", "description": desc,
       "source": "ncu --set full --clock-control none --import-source on (%s)" % rep, "metrics": m}
if alg and "dram__bytes_read.sum" in m:
    def to_b(x):
        u = x["unit"].lower(); v = x["value"]
        return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
    dram = to_b(m["dram__bytes_read.sum"]) + to_b(m["dram__bytes_write.sum"])
    out["algorithmic_bytes"] = alg
    out["dram_bytes_total"] = dram
    out["dram_over_algorithmic"] = dram / alg
print(json.dumps(out, indent=1))
