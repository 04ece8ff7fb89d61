for r in 2 4 8; do
GSV_COMPOSITE_ROWS=$r timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_rows$r.csv python tools/ncu_driver.py 0 > /dev/null 2>&1
GSV_COMPOSITE_ROWS=$r timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 > gpurun_out/bench_rows$r.json 2>/dev/null
done
timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 --streams 16 > gpurun_out/bench_s16.json 2>/dev/null
timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 --streams 4 > gpurun_out/bench_s4.json 2>/dev/null
