# round-2 pass d: in-situ range-decoder profile per channel (run order, runs
# per warp), drop-in suite, 29/30-plane test, codec-1 e2e
set -x
mkdir -p gpurun_out/r2d
timeout 900 python tools/rc_prof.py "" GSV_RC_ORDER=0 GSV_RC_RPW=16 GSV_RC_RPW=8 GSV_RC_RPW=4 GSV_RC_VARIANT=3 > gpurun_out/r2d/rc_prof.log 2>&1
timeout 1200 python -m pytest tests/test_dropin_reference.py tests/test_gpu_scale.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2d/pytest.log 2>&1
timeout 900 python bench.py --codec 1 --no-sweep --sub none --no-cpu --steps 3 --warmup 3 > gpurun_out/r2d/bench_c1.json 2> gpurun_out/r2d/bench_c1.err
