for r in 16384 24576 32768 49152 16384,65536 24576,98304; do
  GSV_ROUNDS=$r timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 > gpurun_out/rounds_$r.json 2>/dev/null
done
