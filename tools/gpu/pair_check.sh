# first GPU run of the CTA-pair scoring kernel: small shapes against the oracle (each
# under its own timeout in case the pair protocol deadlocks), then the pytest subset
set -u
for spec in C5,600 C5,3000 C5,20000 2000,768,300,cosine 3000,512,1000,sqeuclid 1000,256,700,cosine 517,320,513,sqeuclid; do
  timeout 120 python tools/dbg_shapes.py $spec >> gpurun_out/pair_dbg.log 2>&1; echo "$spec rc=$?" >> gpurun_out/pair_dbg.log
  FSIL_TC_PAIR=0 timeout 120 python tools/dbg_shapes.py $spec >> gpurun_out/pair_dbg_off.log 2>&1
done
