set -x
mkdir -p gpurun_out/r2k
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "variants or conformance or truncated or codec or payload" > gpurun_out/r2k/pytest_rc.log 2>&1
timeout 900 python tools/rc_prof.py GSV_RC_SKIP=1 GSV_RC_VARIANT=6,GSV_RC_SKIP=1 "" > gpurun_out/r2k/rc_prof.log 2>&1
