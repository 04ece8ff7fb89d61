python tools/rc_bench.py --planes 3 1 2 > gpurun_out/rcb3.log 2>&1
for v in 1 2; do GSV_RC_VARIANT=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:rc_decode -c 2 -o gpurun_out/rcv$v python tools/rc_bench.py --planes 3 $v > gpurun_out/rcv$v.log 2>&1; done
