"""Per-source-line executed instructions and stall samples of one kernel in an
ncu report (scratch tool): python tools/ncu_inst.py REP KERNEL_SUBSTR [N]."""
import csv, subprocess, sys
rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass,cuda", "--csv"],
                     capture_output=True, text=True).stdout.splitlines()
cur_file, func, hdr = "", "", None
agg = {}
tot_i = tot_s = 0.0
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        func = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or ksub not in func or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    try:
        ie = float(d.get("Instructions Executed") or 0)
        ss = float(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    tot_i += ie; tot_s += ss
    agg[(cur_file, r[0], r[1][:80])] = (ie, ss)
print(f"total {tot_i/1e6:.2f}M warp instructions, {tot_s:.0f} stall samples")
for (f, ln, src), (ie, ss) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{ie/1e6:7.3f}M {100*ss/max(tot_s,1):5.1f}%  {f}:{ln} {src.strip()}")
