set -u
for spec in C5,3000 C5,20000 2000,768,300,cosine 3000,512,1000,sqeuclid 517,320,513,sqeuclid 30000,136,513,sqeuclid 9000,320,2100,cosine; do
  timeout 120 python tools/dbg_shapes.py $spec >> gpurun_out/b2.log 2>&1
done
for cfg in "3 3" "4 2"; do
  set -- $cfg
  FSIL_TC_PAIR_NS=$1 FSIL_TC_PAIR_NB=$2 timeout 300 python tools/perf.py C5:8000000 --reps 2 --out gpurun_out/b2_$1$2.json 2>&1 | tail -1 | cut -c1-300 >> gpurun_out/b2.log
done
