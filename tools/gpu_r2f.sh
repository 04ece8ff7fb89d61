set -x
mkdir -p gpurun_out/r2f
timeout 900 python tools/rc_prof.py GSV_RC_VARIANT=5 > gpurun_out/r2f/rc_prof.log 2>&1
GSV_RC_VARIANT=5 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rc_decode -c 1 -o gpurun_out/r2f/full_rc_decode_v5 python tools/ncu_c2.py 1 > gpurun_out/r2f/full_rc_decode.log 2>&1
