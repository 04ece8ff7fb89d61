# The ncu launch list of the bench command itself (B200_PROFILING.md launch pass;
# per-launch times are cold-cache and serialised: shares, not absolutes).
set -x
O=gpurun_out/prof3
mkdir -p $O
python bench.py --steps 1 --warmup 3 --no-sweep --sub none --no-e2e --no-cpu > /dev/null 2>&1   # inputs cached
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-sweep --sub none --no-e2e --no-cpu > $O/bench_under_ncu.log 2>&1
python tools/launch_summary.py $O/launches_bench.csv > $O/launches_bench_summary.txt 2>&1
gzip -f $O/launches_bench.csv
ls -la $O
