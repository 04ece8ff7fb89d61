set -x
mkdir -p gpurun_out/r2j
GSV_RC_SKIP=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rc_decode -c 1 -o gpurun_out/r2j/rc_u16_only python tools/ncu_c2.py 1 > gpurun_out/r2j/ncu.log 2>&1
