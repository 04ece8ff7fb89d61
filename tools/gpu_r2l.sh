set -x
mkdir -p gpurun_out/r2l
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "variants or conformance or truncated or codec or payload" > gpurun_out/r2l/pytest_rc.log 2>&1
GSV_RC_U8_SPEC=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "variants or conformance or truncated or codec or payload" > gpurun_out/r2l/pytest_rc_u8.log 2>&1
timeout 900 python tools/rc_prof.py "" GSV_RC_SKIP=1 GSV_RC_VARIANT=6,GSV_RC_SKIP=1 GSV_RC_U8_SPEC=2,GSV_RC_SKIP=2 GSV_RC_U8_SPEC=2 > gpurun_out/r2l/rc_prof.log 2>&1
