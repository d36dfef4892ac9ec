"""Per-kernel DRAM traffic per decode step from an ncu launch list.

    python tools/ncu_traffic.py gpurun_out/launches_c4.csv profiles/r02_ncu_traffic.json

The CSV is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` over bench.py --profile-only.  One decode step
launches the update kernel once (the split runs the other kernels once per
session group), so per-step figures are sums over the decode launches divided
by the number of update launches.  ncu serialises and cold-starts every
launch: use the bytes, and only the SHARE of the times."""
import csv
import json
import sys
from collections import defaultdict

NAMES = {"lfps_gate_kernel": "gate", "lfps_stats_kernel": "stats", "lfps_select_kernel": "select",
         "lfps_finish_kernel": "finish", "lfps_update_kernel": "update"}


def main(src, dst):
    rows = [r for r in csv.DictReader(l for l in open(src) if not l.startswith("=="))]
    acc = defaultdict(lambda: defaultdict(float))
    for r in rows:
        name = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]
        key = NAMES.get(name)
        if key is None:
            continue
        v = float(r["Metric Value"].replace(",", ""))
        acc[key][r["Metric Name"]] += v
        if r["Metric Name"] == "gpu__time_duration.sum":
            acc[key]["launches"] += 1
    steps = int(acc["update"]["launches"])
    out = {"source": src, "steps": steps, "kernels": {}}
    for k, a in acc.items():
        rd, wr = a["dram__bytes_read.sum"], a["dram__bytes_write.sum"]
        out["kernels"][k] = {"traffic_bytes": (rd + wr) / steps, "read_bytes": rd / steps,
                             "write_bytes": wr / steps,
                             "ncu_time_ms": a["gpu__time_duration.sum"] / steps / 1e6,
                             "launches_per_step": a["launches"] / steps}
    tot = sum(v["ncu_time_ms"] for v in out["kernels"].values())
    for v in out["kernels"].values():
        v["time_share"] = v["ncu_time_ms"] / tot
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:3])
