set -x
O=gpurun_out/r2ae
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sequence.py -q -p no:cacheprovider -rf > $O/pytest_seq.log 2>&1
timeout 1500 python bench.py --sub none --no-sweep > $O/bench.json 2> $O/bench.err
GSV_VALUE_SEQ=0 timeout 1500 python bench.py --sub none --no-sweep --no-e2e --no-cpu > $O/bench_oldvalue.json 2> $O/bench_oldvalue.err
