"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per
kernel launch of the last N launches (scratch analysis tool)."""
import collections, csv, sys
path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {h: i for i, h in enumerate(hdr)}
agg = collections.OrderedDict()
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    name = r[ix["Kernel Name"]].split("(")[0].split("::")[-1]
    val = float(r[ix["Metric Value"]].replace(",", ""))
    agg.setdefault((int(r[ix["ID"]]), name), {})[r[ix["Metric Name"]]] = val
tot = 0.0
for (i, name), m in list(agg.items())[-last:]:
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    rd = m.get("dram__bytes_read.sum", 0) / 1e9
    wr = m.get("dram__bytes_write.sum", 0) / 1e9
    tot += t
    bw = (rd + wr) / (t * 1e-6) if t else 0
    print(f"{i:>6} {name[:36]:36s} {t:9.1f} us  rd {rd:7.3f} GB  wr {wr:7.3f} GB  {bw:6.0f} GB/s")
print(f"sum {tot:.1f} us")
