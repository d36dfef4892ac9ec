"""Per-CUDA-source-line warp-stall summary of an ncu report (scratch tool)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass,cuda", "--csv"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
cur_file = ""
lines = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] != "":
        ix = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            samples = int(r[ix] or 0)
        except (ValueError, IndexError):
            continue
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        best = max(stall_cols, key=lambda i: int(r[i] or 0)) if stall_cols else None
        lines.append((samples, cur_file, r[0], r[1].strip()[:70], hdr[best][6:] if best else ""))
tot = sum(l[0] for l in lines) or 1
lines.sort(key=lambda x: -x[0])
for s, f, ln, src, st in lines[:top]:
    print(f"{s/tot:6.1%} {f}:{ln:>4} {st:14s} {src}")
