# full-size parity tests (C3, C4 all rows vs the oracle; C5 fast vs fp64 path + oracle rows)
timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "full_size" > gpurun_out/fullsize.log 2>&1
echo "fullsize rc=$?" >> gpurun_out/fullsize.log
