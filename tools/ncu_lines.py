"""Per-CUDA-source-line instruction counts and stall samples from an ncu source page.

    ncu -i rep --page source --csv --print-source cuda,sass [-k name] | python tools/ncu_lines.py [N]
"""
import csv
import sys

N = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rows = list(csv.reader(sys.stdin))
data = {}
files = {}
cur_file = None
first_fn = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        if first_fn is None:
            first_fn = r[1]
        elif r[1] != first_fn:
            break
        continue
    if r[0] == "Line No":
        hdr = r
        I = hdr.index("Instructions Executed")
        S = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or r[0] == "":
        continue
    try:
        n = int(r[I] or 0)
        s = int(r[S] or 0)
    except ValueError:
        continue
    key = (cur_file, int(r[0]))
    d = data.setdefault(key, [0, 0, r[1][:90]])
    d[0] += n
    d[1] += s
tot = sum(v[0] for v in data.values()) or 1
ts = sum(v[1] for v in data.values()) or 1
print(first_fn, "total warp-inst", tot)
for k, v in sorted(data.items(), key=lambda kv: -kv[1][0])[:N]:
    print("%10d %5.1f%% st %5.1f%%  %s:%d  %s" % (v[0], 100 * v[0] / tot, 100 * v[1] / ts, k[0], k[1], v[2]))
print("--- by stall samples")
for k, v in sorted(data.items(), key=lambda kv: -kv[1][1])[:N]:
    print("%10d %5.1f%% st %5.1f%%  %s:%d  %s" % (v[0], 100 * v[0] / tot, 100 * v[1] / ts, k[0], k[1], v[2]))
