# Round-2 profile artefacts (one GPU): launch lists of a config-2 open +
# 4 rendered frames for codec 0 and codec 1, one ncu --set full capture of
# every stage kernel on the full 300-frame config-2 container (CRC and range
# decode of the whole sequence, then the per-frame render kernels), the
# one-pass motion fold, and a stage table.  Reports are summarised on the box
# (text/CSV) and only the compositor's report is kept (gpurun copies back at
# most 64 MiB).
set -x
O=gpurun_out/prof2
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_codec0.csv python tools/ncu_c2.py 0 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_codec1.csv python tools/ncu_c2.py 1 > /dev/null 2>&1
K='crc_kernel|project_kernel|depth_key_prep|radix_onesweep|depth_tie_fixup|r1_count|r1_scan_blocks|r1_scan_tiles|r1_place|round_emit_fused|keys_to_off|open_mask|composite_strip|reset_frame'
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 40 -o $O/full_c2_codec0 python tools/ncu_c2.py 0 > $O/full_c2_codec0.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"rc_decode|copy_planes|crc_kernel" -c 3 -o $O/full_c2_codec1_open python tools/ncu_c2.py 1 > $O/full_c2_codec1_open.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fold -s 1 -c 1 -o $O/full_fold python tools/fold_driver.py > $O/full_fold.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:composite_strip -c 2 -o $O/composite python tools/ncu_c2.py 0 > $O/composite.log 2>&1
for r in $O/full_*.ncu-rep $O/composite.ncu-rep; do
  python tools/ncu_summary.py $r > ${r%.ncu-rep}_summary.txt 2>&1
done
ncu -i $O/composite.ncu-rep --page source --csv --print-source sass > $O/composite_source.csv 2>/dev/null
python tools/stage_table.py $O > $O/stage_table.md 2>&1
rm -f $O/full_*.ncu-rep
ls -la $O
du -sh gpurun_out
