"""Summarise an ncu report's SASS source page: hottest instructions by warp
stall samples, with executed-instruction counts (scratch analysis tool)."""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[1:]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
inst = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
print(f"total stall samples {tot}, instructions executed {inst}")
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {c: 0 for c in stall_cols}
for r in data:
    for c in stall_cols:
        agg[c] += int(r[ix[c]] or 0)
print("stall mix:", ", ".join(f"{c[6:]}={v/tot:.1%}" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for r in data[:top]:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top_stall = max(stall_cols, key=lambda c: int(r[ix[c]] or 0))
    print(f"{s/tot:6.1%} {int(r[ix['Instructions Executed']] or 0):>11} {r[ix['Address']][-5:]} "
          f"{r[ix['Source']].strip()[:60]:60s} {top_stall[6:]}")
