"""Hottest SASS lines of one kernel in an ncu report (source page).
python tools/ncu_sass_hot.py rep.ncu-rep <kernel index> [top]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for row in csv.reader(io.StringIO(out)):
    if row and row[0] == "Kernel Name":
        cur = {"name": row[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(row)
b = blocks[idx]
hdr = b["rows"][0]
recs = [dict(zip(hdr, r)) for r in b["rows"][1:]]
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in recs)
print(b["name"][:120], "samples", tot, "instructions", len(recs))
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {s: sum(int(r[s] or 0) for r in recs) for s in stalls}
print("  ", "  ".join(f"{k[6:]}={v}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v))
for r in sorted(recs, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    top_st = sorted(((int(r[k] or 0), k[6:]) for k in stalls), reverse=True)[:2]
    print(f"{s:6d} {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} {top_st}")
