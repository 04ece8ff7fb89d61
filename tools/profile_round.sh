# Round profile artefacts (one GPU): launch lists for codec 0 and 1, ncu --set
# full captures of the top kernels, and one full bench line.
mkdir -p gpurun_out/prof
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_codec0.csv python tools/ncu_driver.py 0 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_codec1.csv python tools/ncu_driver.py 1 > /dev/null 2>&1
for k in composite_strip radix_onesweep round_emit_fused project_kernel r1_place r1_count depth_tie_fixup crc_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 2 \
     -o gpurun_out/prof/full_$k python tools/ncu_driver.py 0 > gpurun_out/prof/full_$k.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rc_decode -c 1 \
     -o gpurun_out/prof/full_rc_decode python tools/rc_bench.py --planes 3 3 > gpurun_out/prof/full_rc_decode.log 2>&1
ENC_N=50000 ENC_FRAMES=30 ENC_SKIP_HOST=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:rc_encode -c 1 \
     -o gpurun_out/prof/full_rc_encode python tools/enc_bench.py > gpurun_out/prof/full_rc_encode.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fold -s 1 -c 1 \
     -o gpurun_out/prof/full_fold python tools/fold_driver.py > gpurun_out/prof/full_fold.log 2>&1
