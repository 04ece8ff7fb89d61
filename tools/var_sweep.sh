# dev: bench a list of env-var variants: VARIANTS="name:ENV=V,ENV2=V2 ..."
for spec in $VARIANTS; do
  name=${spec%%:*}; envs=${spec#*:}
  env $(echo $envs | tr ',' ' ') timeout 900 python bench.py --no-sweep --no-cpu --no-e2e --steps 3 > gpurun_out/var_$name.json 2>/dev/null
done
