# dev diagnostic: marginal cost of each stage in the frame-parallel steady
# state -- the stage is launched twice (idempotent stages only), the extra
# ms per step is its marginal cost
for st in ${STAGES:-none composite tsort dsort emit project fixup lastround}; do
  GSV_DEBUG_DOUBLE=$st timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --sub none --steps 5 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$st', d['value'], d['ms_per_step'])"
done
