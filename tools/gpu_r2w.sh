set -x
O=gpurun_out/r2w
mkdir -p $O
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python tools/e2e_probe.py > $O/e2e_probe_conn32.txt 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=16 timeout 900 python tools/e2e_probe.py > $O/e2e_probe_conn16.txt 2>&1
