set -x
O=gpurun_out/r2al
mkdir -p $O
timeout 1200 python tools/composite_ab.py "GSV_R1_PLACE=1" "GSV_R1_PLACE=2" "GSV_R1_PLACE=1" "GSV_R1_PLACE=2" > $O/ab.txt 2>&1
rm -rf gpurun_out/ab
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -p no:cacheprovider -rf -k "identically or c5 or c2_projection or ring or tie" > $O/pytest.log 2>&1
timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --sub none > $O/bench.json 2> $O/bench.err
