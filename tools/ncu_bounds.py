"""What bounds each kernel of an ncu --set full report: issue activity,
occupancy, DRAM / L2 / L2->SM throughput, the busiest pipe and the top warp
stall reasons per issued instruction.

    python tools/ncu_bounds.py gpurun_out/ev/prof_c4.ncu-rep > profiles/r02_c4_ncu_bounds.txt
"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def f(d, k):
        try:
            return float(d.get(k, "nan"))
        except ValueError:
            return float("nan")
    print("# per kernel: time, warp-instructions, issue-active %, warps-active %, DRAM %, "
          "L2 (lts) %, L2->SM bytes and % of peak, busiest pipe %, top stalls "
          "(cycles per issued instruction)")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = r[4].split("(")[0].replace("unnamed>::", "")
        pipes = {k.split("__")[1].split(".")[0]: f(d, k) for k in d
                 if k.startswith("sm__pipe_") and k.endswith("cycles_active.avg.pct_of_peak_sustained_active")}
        pipes.update({k.split("__")[1].split(".")[0]: f(d, k) for k in d
                      if k.startswith("sm__inst_executed_pipe_")
                      and k.endswith(".avg.pct_of_peak_sustained_active")})
        busiest = max(pipes.items(), key=lambda kv: kv[1] if kv[1] == kv[1] else -1) if pipes else ("-", 0)
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(d, k)
                  for k in d if k.startswith("smsp__average_warps_issue_stalled_")
                  and k.endswith("_per_issue_active.ratio")}
        top = sorted(((v, k) for k, v in stalls.items() if v == v), reverse=True)[:5]
        print(f"{name:32s} {f(d, 'gpu__time_duration.sum'):8.1f} us  "
              f"inst {f(d, 'smsp__inst_executed.sum') / 1e6:6.1f} M  "
              f"issue {f(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):4.1f}%  "
              f"warps {f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):4.1f}%  "
              f"dram {f(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):4.1f}%  "
              f"lts {f(d, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):4.1f}%  "
              f"L2->SM {f(d, 'l1tex__m_xbar2l1tex_read_bytes.sum') * scale.get(units.get('l1tex__m_xbar2l1tex_read_bytes.sum'), 1.0) / 1e6:7.1f} MB "
              f"({f(d, 'l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed'):4.1f}%)  "
              f"pipe {busiest[0]} {busiest[1]:4.1f}%  "
              f"stalls " + ", ".join(f"{k} {v:.2f}" for v, k in top))


if __name__ == "__main__":
    main()
