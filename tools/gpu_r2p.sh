# Round-2 profiles + step diagnostics + range-decoder per-run profile.
set -x
O=gpurun_out/r2p
mkdir -p $O
timeout 600 python tools/step_diag.py 0 > $O/step_diag_c0.txt 2>&1
GSV_DEBUG_OPEN_TIMING=1 timeout 300 python tools/step_diag.py 0 > $O/step_diag_c0_timing.txt 2>&1
timeout 900 python tools/rc_prof.py "" > $O/rc_prof.txt 2>&1
timeout 3000 bash tools/profile_round2.sh > $O/prof.log 2>&1
du -sh gpurun_out/*
