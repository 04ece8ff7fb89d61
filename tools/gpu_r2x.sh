set -x
O=gpurun_out/r2x
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sequence.py -q -p no:cacheprovider -rf > $O/pytest_seq.log 2>&1
timeout 900 python tools/e2e_probe.py > $O/e2e_probe.txt 2>&1
timeout 900 python tools/composite_ab.py "GSV_COMPOSITE_PACKED=2" "GSV_COMPOSITE_PACKED=3,GSV_COMPOSITE_MINB=5" "GSV_COMPOSITE_PACKED=3,GSV_COMPOSITE_MINB=4" > $O/ab.txt 2>&1
rm -rf gpurun_out/ab
