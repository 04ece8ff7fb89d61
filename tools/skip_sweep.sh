# dev diagnostic: frame-parallel throughput with stages skipped (images invalid)
for sk in ${SKIPS:-none composite tsort dsort emit project gather fixup}; do
  GSV_DEBUG_SKIP=$sk timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sk', d['value'], d['ms_per_step'])"
done
