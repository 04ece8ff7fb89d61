# Round-2 re-entry check: full GPU test suite, default bench line, round-2 profiles.
set -x
mkdir -p gpurun_out/r2n
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2n/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2n/pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/r2n/bench.json 2> gpurun_out/r2n/bench.err
timeout 3000 bash tools/profile_round2.sh > gpurun_out/r2n/prof.log 2>&1
