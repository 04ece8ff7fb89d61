# round-2 first GPU pass: smoke, all GPU tests, a quick bench line, ncu of the
# config-2 codec-1 range decoder launch (all 1380 runs) and the CRC kernel.
set -x
mkdir -p gpurun_out/r2a
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2a/pytest.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2a/launches_c2_codec1.csv python tools/ncu_c2.py 1 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rc_decode -c 1 -o gpurun_out/r2a/full_rc_decode_c2 python tools/ncu_c2.py 1 > gpurun_out/r2a/full_rc_decode.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:crc_kernel -c 1 -o gpurun_out/r2a/full_crc_c2 python tools/ncu_c2.py 0 > gpurun_out/r2a/full_crc.log 2>&1
ls -la gpurun_out/r2a
