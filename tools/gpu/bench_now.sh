set -u
timeout 1200 python bench.py > gpurun_out/bench_r02b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r02b.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_r02b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_r02b.log
