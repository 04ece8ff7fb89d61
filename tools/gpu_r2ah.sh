set -x
O=gpurun_out/r2ah
mkdir -p $O
timeout 1200 python tools/composite_ab.py "GSV_COMPOSITE_CFG=0" "GSV_COMPOSITE_CFG=1" "GSV_COMPOSITE_CFG=2" "GSV_COMPOSITE_CFG=0" "GSV_COMPOSITE_CFG=1" "GSV_COMPOSITE_CFG=2" > $O/ab.txt 2>&1
rm -rf gpurun_out/ab
