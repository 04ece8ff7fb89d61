set -x
O=gpurun_out/r2ak
mkdir -p $O
python bench.py --no-sweep --no-cpu --no-e2e --sub none --steps 2 --warmup 3 > /dev/null 2>&1
STAGES="none r1count r1place composite none" bash tools/double_sweep.sh > $O/double_sweep.txt 2>&1
