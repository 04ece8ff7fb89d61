# Round-2: compositor V3 A/B, full GPU test suite, default bench line.
set -x
O=gpurun_out/r2o
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 900 python tools/composite_ab.py "GSV_COMPOSITE_PACKED=2" "GSV_COMPOSITE_PACKED=3,GSV_COMPOSITE_MINB=5" "GSV_COMPOSITE_PACKED=3,GSV_COMPOSITE_MINB=4" "GSV_COMPOSITE_PACKED=2" > $O/ab.txt 2>&1
rm -rf gpurun_out/ab
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
du -sh gpurun_out
