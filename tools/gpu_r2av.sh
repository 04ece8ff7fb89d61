set -x
O=gpurun_out/r2av
mkdir -p $O
timeout 1200 python tools/composite_ab.py "GSV_COMPOSITE_PACKED=4" "GSV_COMPOSITE_PACKED=5" "GSV_COMPOSITE_PACKED=4" "GSV_COMPOSITE_PACKED=5" > $O/ab.txt 2>&1
rm -rf gpurun_out/ab
