set -x
O=gpurun_out/r2aj
mkdir -p $O
timeout 1200 python tools/composite_ab.py "" "GSV_PROJ_REGS=72" "GSV_PROJ_REGS=64" "" > $O/ab_proj.txt 2>&1
rm -rf gpurun_out/ab
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1
