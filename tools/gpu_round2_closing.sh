# Round-2 closing run: full GPU test suite, default bench line, reference arm, 2-rank check, profiles.
set -x
O=gpurun_out/final2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-sweep --sub none --no-cpu > $O/bench_2ranks.json 2> $O/bench_2ranks.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 3000 bash tools/profile_round2.sh > $O/prof.log 2>&1
du -sh gpurun_out/*
