# compute-sanitizer over the decode path (incl. the stream split), then the
# C1 / C2 / C3 bench lines
set -x
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo $tool rc $?
  tail -3 gpurun_out/sanitize_$tool.log
done
for cfg in c1 c2; do
  timeout 600 python bench.py --config $cfg --no-cpu > gpurun_out/bench_$cfg.log 2>&1; echo $cfg rc $?
  tail -1 gpurun_out/bench_$cfg.log | cut -c1-400
done
timeout 900 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo c3 rc $?
tail -1 gpurun_out/bench_c3.log | cut -c1-300
