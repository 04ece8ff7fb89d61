set -x
mkdir -p gpurun_out/r2g
timeout 1200 python tools/rc_prof.py GSV_RC_VARIANT=4 "" GSV_RC_SKIP=1 GSV_RC_U8_SPEC=1,GSV_RC_SKIP=2 GSV_RC_SKIP=2 GSV_RC_U8_SPEC=1 > gpurun_out/r2g/rc_prof.log 2>&1
