# compute-sanitizer over smoke() + a config-1 decode/render.
# Outputs: gpurun_out/sanitize/{memcheck,racecheck,synccheck,initcheck}.log
O=gpurun_out/sanitize
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_driver.py > $O/$tool.log 2>&1
  echo "$tool exit $?" >> $O/summary.txt
done
