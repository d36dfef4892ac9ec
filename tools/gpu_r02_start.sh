# Session start: GPU parity suite at HEAD, then the round-2 evidence script.
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ev/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/ev/gputests.txt 2>&1; echo "gpu tests rc $?"
tail -3 gpurun_out/ev/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.txt 2>&1; echo "smoke rc $?"
bash tools/gpu_evidence_r02.sh
