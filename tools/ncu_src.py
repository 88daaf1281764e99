"""Summarise an ncu source page (SASS) of one kernel: instruction mix and stall reasons.

    ncu -i rep --page source --csv --print-source sass -k <kernel> | python tools/ncu_src.py
"""
import collections
import csv
import sys

rows = list(csv.reader(sys.stdin))
kern = None
blocks = []
cur = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
        hdr = None
        continue
    if r and r[0] == "Address":
        cur["hdr"] = r
        continue
    if cur is not None and "hdr" in cur and r:
        cur["rows"].append(r)
for b in blocks[:1]:
    h = b["hdr"]
    I = h.index("Instructions Executed")
    S = h.index("Warp Stall Sampling (All Samples)")
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    si = [h.index(c) for c in stalls]
    mix = collections.Counter()
    st = collections.Counter()
    tot = 0
    for r in b["rows"]:
        src = r[1].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        n = int(r[I] or 0)
        mix[op] += n
        tot += n
        for c, i in zip(stalls, si):
            st[c] += int(r[i] or 0)
    print(b["name"][:100], "total warp-inst", tot)
    for op, n in mix.most_common(30):
        print("  %-10s %12d %5.1f%%" % (op, n, 100.0 * n / tot))
    ts = sum(st.values())
    print("stalls:")
    for c, n in st.most_common(12):
        print("  %-22s %5.1f%%" % (c, 100.0 * n / ts))
