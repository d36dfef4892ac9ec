# final bench lines at HEAD: C4 (with the stock-reference cpu_baseline), C1, C2, C3 and the per-rank C4 shares
set -x
mkdir -p gpurun_out/fin
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin/c4.jsonl 2> gpurun_out/fin/c4.err
timeout 600 python bench.py --config c1 --steps 50 --warmup 5 > gpurun_out/fin/c1.jsonl 2> gpurun_out/fin/c1.err
timeout 600 python bench.py --config c2 --steps 50 --warmup 5 > gpurun_out/fin/c2.jsonl 2> gpurun_out/fin/c2.err
for c in c4s2 c4s4 c4s8; do timeout 600 python bench.py --config $c --no-cpu --steps 30 --warmup 5 > gpurun_out/fin/$c.jsonl 2> gpurun_out/fin/$c.err; done
timeout 1500 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/fin/c3.jsonl 2> gpurun_out/fin/c3.err
for f in c4 c1 c2 c3; do tail -c 200 gpurun_out/fin/$f.err; done
