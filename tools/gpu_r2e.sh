# round-2 pass e: variant 5 (warp-cooperative speculative range decoder)
set -x
mkdir -p gpurun_out/r2e
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "variants or conformance or truncated or codec or payload" > gpurun_out/r2e/pytest_rc.log 2>&1
timeout 900 python tools/rc_prof.py GSV_RC_VARIANT=4 GSV_RC_VARIANT=5 > gpurun_out/r2e/rc_prof.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2e/pytest.log 2>&1
timeout 900 python bench.py --codec 1 --no-sweep --sub none --no-cpu --steps 3 --warmup 3 > gpurun_out/r2e/bench_c1.json 2> gpurun_out/r2e/bench_c1.err
