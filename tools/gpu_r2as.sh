set -x
O=gpurun_out/r2as
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sequence.py -q -p no:cacheprovider -rf > $O/pytest_seq.log 2>&1
timeout 600 python tools/seq_timeline.py > $O/timeline.txt 2>&1
GSV_SEQ_PLANE_MAJOR=0 timeout 600 python tools/seq_timeline.py > $O/timeline_nopm.txt 2>&1
