set -x
O=gpurun_out/r2aa
mkdir -p $O
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python tools/seq_timeline.py > $O/timeline_c32.txt 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python tools/e2e_probe.py > $O/e2e_probe_c32.txt 2>&1
