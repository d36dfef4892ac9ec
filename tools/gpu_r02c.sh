set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lfps_api.py -q -x 2>&1 | tail -30 > gpurun_out/lfps_api.txt
timeout 1200 python -m pytest tests/test_gpu_reference_suite.py -q -s 2>&1 | tail -150 > gpurun_out/ref_suite.txt
cat gpurun_out/lfps_api.txt | tail -30
grep -E "passed|failed|FAILED|Error" gpurun_out/ref_suite.txt | head -60
