# Round-2: render_sequence v3 (descriptors before payload uploads), compact rect array; tests + diag + bench.
set -x
O=gpurun_out/r2t
mkdir -p $O
timeout 600 python tools/step_diag.py 0 > $O/step_diag_c0.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1
timeout 1500 python bench.py --sub none --no-sweep > $O/bench.json 2> $O/bench.err
