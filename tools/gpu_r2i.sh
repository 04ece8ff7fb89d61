set -x
mkdir -p gpurun_out/r2i
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "variants or conformance or truncated or codec or payload" > gpurun_out/r2i/pytest_rc.log 2>&1
timeout 900 python tools/rc_prof.py "" GSV_RC_SKIP=1 > gpurun_out/r2i/rc_prof.log 2>&1
