set -x
O=gpurun_out/r2ap
mkdir -p $O
timeout 1200 python tools/composite_ab.py "" "GSV_R2_ROWS=4" "GSV_R2_ROWS=2" "" "GSV_R2_ROWS=4" "GSV_R2_ROWS=2" > $O/ab.txt 2>&1
rm -rf gpurun_out/ab
