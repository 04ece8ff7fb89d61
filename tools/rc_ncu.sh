# ncu source-level captures of the range decoder (dev tool): launches 3-4 are the 16-bit run
python tools/rc_bench.py --planes 3 2 3 > gpurun_out/rcb3.log 2>&1
for v in ${RC_VARIANTS:-2 3}; do GSV_RC_VARIANT=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:rc_decode -c 4 -o gpurun_out/rcv$v python tools/rc_bench.py --planes 3 $v > gpurun_out/rcv$v.log 2>&1; done
