# compute-sanitizer over every libfsil kernel variant (tools/sanitize_cases.py), small N.
# ONE tool per gpurun call (B200_PROFILING.md): bash tools/gpu/sanitize.sh memcheck|racecheck|synccheck|initcheck
# The cases first run plain (must exit 0) before the sanitizer touches them.
set -u
tool=$1
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_cases.py > gpurun_out/san_plain_$tool.log 2>&1 || { echo "plain run failed" >> gpurun_out/san_plain_$tool.log; exit 1; }
extra=""
[ "$tool" = memcheck ] && extra="--leak-check full"
timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
    python tools/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
echo "$tool rc=$?" >> gpurun_out/san_$tool.log
