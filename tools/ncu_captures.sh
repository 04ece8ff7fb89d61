# ncu --set full captures of the top kernels (one GPU; dev tool).
# usage: bash tools/ncu_captures.sh <tag> [kernels...]
tag=${1:-cap}; shift
ks=${@:-"composite_round_kernel rc_decode_kernel project_kernel round_emit_fused radix_downsweep"}
mkdir -p gpurun_out
for k in $ks; do
  case $k in
    rc_decode_kernel) cod=1; cnt=2;;
    *) cod=0; cnt=2;;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-2} -c $cnt \
     -o gpurun_out/${tag}_$k python tools/ncu_driver.py $cod > gpurun_out/${tag}_$k.log 2>&1
done
