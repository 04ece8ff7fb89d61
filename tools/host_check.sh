for sk in none composite,tsort,dsort,emit; do
  GSV_DEBUG_SKIP=$sk timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 > gpurun_out/host_$sk.json 2>/dev/null
done
