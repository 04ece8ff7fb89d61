set -x
mkdir -p gpurun_out/r2m
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2m/pytest.log 2>&1
GSV_RC_U8_SPEC=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "variants" > gpurun_out/r2m/pytest_u8m0.log 2>&1
GSV_RC_U8_SPEC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "variants" > gpurun_out/r2m/pytest_u8m1.log 2>&1
timeout 1200 python bench.py > gpurun_out/r2m/bench.json 2> gpurun_out/r2m/bench.err
