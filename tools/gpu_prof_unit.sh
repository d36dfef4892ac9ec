# ncu: launch list + one --set full capture of the select / finish kernels at C4
mkdir -p gpurun_out/pu
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --verify 0 > gpurun_out/pu/c4.jsonl 2> gpurun_out/pu/c4.err; echo "c4 rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"lfps_(gate|stats|select|finish|unit|update)" -s 12 -c 12 --csv --log-file gpurun_out/pu/launches.csv \
  python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/pu/ncu_list.log 2>&1; echo list rc $?
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"lfps_(select|unit|finish)" -s 6 -c 2 -o gpurun_out/pu/prof_c4 -f \
  python bench.py --profile-only --steps 2 --warmup 2 > gpurun_out/pu/ncu_full.log 2>&1; echo full rc $?
python tools/ncu_summary.py gpurun_out/pu/prof_c4.ncu-rep > gpurun_out/pu/summary.txt 2>&1
cat gpurun_out/pu/summary.txt
python - <<'PY'
import json
for l in open("gpurun_out/pu/c4.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["value"], d.get("kernel_ms"))
PY
