# per-unit finish A/B: parity of the unit tests, then C4 lines (session finish,
# unit finish on the default build and on variant libraries)
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests -m gpu -x -q -k "unit_finish" > gpurun_out/ab/tests.txt 2>&1; echo "tests rc $?"; tail -2 gpurun_out/ab/tests.txt
line() { python -c "import json,sys
for l in open('$1'):
    if l.startswith('{'): d=json.loads(l); print('$2', round(d['value'],1), {k: round(v*1000,1) for k,v in d['kernel_ms'].items()})"; }
timeout 300 python bench.py --no-cpu --verify 0 --steps 20 > gpurun_out/ab/sess.jsonl 2>/dev/null; line gpurun_out/ab/sess.jsonl session
timeout 300 python bench.py --no-cpu --verify 1 --steps 20 --unit-finish > gpurun_out/ab/unit.jsonl 2>gpurun_out/ab/unit.err; line gpurun_out/ab/unit.jsonl unit-default
for v in ${VARIANTS:-}; do
  LFPS_LIB=$PWD/paper_2506_15704_b200/lib/variants/$v.so timeout 300 python bench.py --no-cpu --verify 0 --steps 20 --unit-finish > gpurun_out/ab/$v.jsonl 2>/dev/null; line gpurun_out/ab/$v.jsonl unit-$v
done
tail -3 gpurun_out/ab/unit.err
