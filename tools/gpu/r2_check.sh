set -u
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 ) > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
