# ncu source-level capture of the GPU range coder (dev tool)
ENC_N=50000 ENC_FRAMES=30 ENC_SKIP_HOST=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:rc_encode -c 1 -o gpurun_out/enc python tools/enc_bench.py > gpurun_out/enc_ncu.log 2>&1
