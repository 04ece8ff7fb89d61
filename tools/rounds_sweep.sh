# depth-rank round boundaries sweep (dev tool): GSV_ROUNDS = absolute ranks
for r in ${ROUNDS:-16384 24576 32768 49152 65536 16384,65536 32768,131072}; do
  GSV_ROUNDS=$r timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$r', d['value'], d['stages_ms_per_frame']['composite'], d['render_stats']['n_keys_emitted'])"
done
