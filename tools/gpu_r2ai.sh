set -x
O=gpurun_out/r2ai
mkdir -p $O
timeout 1200 python tools/composite_ab.py "GSV_COMPOSITE_PACKED=3" "GSV_COMPOSITE_PACKED=4" "GSV_COMPOSITE_PACKED=3" "GSV_COMPOSITE_PACKED=4" > $O/ab.txt 2>&1
rm -rf gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -rf -k "variants or identically or conformance" > $O/pytest.log 2>&1
timeout 1500 compute-sanitizer --tool initcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_driver.py > $O/initcheck.log 2>&1; echo "initcheck exit $?" >> $O/initcheck.log
