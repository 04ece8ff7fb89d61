# Round-2: render_sequence (pipelined e2e) tests + step diag + bench.
set -x
O=gpurun_out/r2r
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sequence.py -q -p no:cacheprovider -rf -x > $O/pytest_seq.log 2>&1
timeout 600 python tools/step_diag.py 0 > $O/step_diag_c0.txt 2>&1
timeout 1500 python bench.py --sub none --no-sweep > $O/bench.json 2> $O/bench.err
