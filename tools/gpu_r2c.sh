# round-2 pass c (re-entry): smoke, all GPU tests incl. the reference-suite drop-in,
# default bench, sharded bench on 2 ranks, ncu of the c2 codec-1 decoder and CRC.
set -x
mkdir -p gpurun_out/r2c
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2c/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=30 > gpurun_out/r2c/pytest.log 2>&1
timeout 1200 python bench.py > gpurun_out/r2c/bench.json 2> gpurun_out/r2c/bench.err
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-sweep --sub none --no-cpu > gpurun_out/r2c/bench_g2.json 2> gpurun_out/r2c/bench_g2.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rc_decode -c 1 -o gpurun_out/r2c/full_rc_decode_c2 python tools/ncu_c2.py 1 > gpurun_out/r2c/full_rc_decode.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:crc_kernel -c 1 -o gpurun_out/r2c/full_crc_c2 python tools/ncu_c2.py 0 > gpurun_out/r2c/full_crc.log 2>&1
ls -la gpurun_out/r2c
