set -x
O=gpurun_out/r2ar
mkdir -p $O
timeout 1500 python tools/composite_ab.py "" "GSV_DEPTH_KEY_BITS=16" "GSV_ROUNDS=24576" "GSV_ROUNDS=40960" "GSV_ROUNDS=49152" "" > $O/ab.txt 2>&1
rm -rf gpurun_out/ab
