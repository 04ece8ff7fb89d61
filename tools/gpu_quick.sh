# quick GPU check: parity tests, codec-1 launch list, short bench (dev tool)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_codec1.csv python tools/ncu_driver.py 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_codec0.csv python tools/ncu_driver.py 0 > /dev/null 2>&1
timeout 1200 python bench.py --no-cpu --steps 3 ${BENCH_ARGS} > gpurun_out/bench.json 2>gpurun_out/bench.err
