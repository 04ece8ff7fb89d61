set -x
O=gpurun_out/r2an
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1
GSV_DEBUG_OPEN_TIMING=1 timeout 600 python tools/step_diag.py 0 > $O/step_diag.txt 2>&1
timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --sub none > $O/bench.json 2> $O/bench.err
