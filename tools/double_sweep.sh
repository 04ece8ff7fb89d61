# dev diagnostic: marginal frame-parallel cost of a stage = throughput drop when it runs twice
for d in none composite dsort tsort project; do
  GSV_DEBUG_DOUBLE=$d timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 > gpurun_out/dbl_$d.json 2>/dev/null
done
