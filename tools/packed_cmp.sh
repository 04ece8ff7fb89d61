timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
for p in 1 0; do
GSV_COMPOSITE_PACKED=$p timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_packed$p.csv python tools/ncu_driver.py 0 > /dev/null 2>&1
GSV_COMPOSITE_PACKED=$p timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 > gpurun_out/bench_packed$p.json 2>/dev/null
done
GSV_COMPOSITE_ROWS=4 timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 > gpurun_out/bench_packed1_r4.json 2>/dev/null
