set -x
O=gpurun_out/r2ab
mkdir -p $O
timeout 600 python tools/seq_timeline.py > $O/timeline.txt 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python tools/seq_timeline.py > $O/timeline_c32.txt 2>&1
