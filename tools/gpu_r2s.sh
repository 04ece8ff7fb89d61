# Round-2: render_sequence v2 (all uploads first) tests + step diag + e2e bench.
set -x
O=gpurun_out/r2s
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sequence.py tests/test_gpu_parity.py -q -p no:cacheprovider -rf > $O/pytest_seq.log 2>&1
timeout 600 python tools/step_diag.py 0 > $O/step_diag_c0.txt 2>&1
timeout 1500 python bench.py --sub none --no-sweep > $O/bench.json 2> $O/bench.err
GSV_E2E_SEQ=0 timeout 1500 python bench.py --sub none --no-sweep --no-cpu > $O/bench_threaded.json 2> $O/bench_threaded.err
