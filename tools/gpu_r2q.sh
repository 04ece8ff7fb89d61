# Round-2: CRC v2 + compositor FULL path A/B, tests, step diagnostics, CRC ncu.
set -x
O=gpurun_out/r2q
mkdir -p $O
timeout 900 python tools/composite_ab.py "GSV_COMPOSITE_PACKED=2" "GSV_COMPOSITE_PACKED=3,GSV_COMPOSITE_MINB=5" "GSV_COMPOSITE_PACKED=3,GSV_COMPOSITE_MINB=4" > $O/ab.txt 2>&1
rm -rf gpurun_out/ab
timeout 600 python tools/step_diag.py 0 > $O/step_diag_c0.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > $O/pytest.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:crc_kernel -c 1 -o $O/crc python tools/ncu_c2.py 0 > $O/crc.log 2>&1
python tools/ncu_summary.py $O/crc.ncu-rep > $O/crc_summary.txt 2>&1
rm -f $O/crc.ncu-rep
