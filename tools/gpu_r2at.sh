set -x
O=gpurun_out/r2at
mkdir -p $O
timeout 1200 python tools/composite_ab.py "GSV_PROJ_WAVES=0" "" "GSV_PROJ_WAVES=2" "GSV_PROJ_WAVES=0" "" "GSV_PROJ_WAVES=2" > $O/ab.txt 2>&1
rm -rf gpurun_out/ab
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -p no:cacheprovider -rf -k "c2_projection or render_matches or edge or acceptance or config1 or tie" > $O/pytest.log 2>&1
