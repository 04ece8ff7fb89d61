# round-2 second pass: new decoder (variant 4) + tie fix-up tail, sharded bench
set -x
mkdir -p gpurun_out/r2b
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_shard.py -m gpu -q -p no:cacheprovider > gpurun_out/r2b/pytest.log 2>&1
timeout 600 python tools/rc_time.py 3 4 > gpurun_out/r2b/rc_time.log 2>&1
timeout 1200 python bench.py > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-sweep --sub none --no-cpu > gpurun_out/r2b/bench_g2.json 2> gpurun_out/r2b/bench_g2.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rc_decode -c 1 -o gpurun_out/r2b/full_rc_decode_v4 python tools/ncu_c2.py 1 > gpurun_out/r2b/full_rc_decode.log 2>&1
ls -la gpurun_out/r2b
