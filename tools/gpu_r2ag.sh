set -x
O=gpurun_out/r2ag
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"project_kernel|composite_strip" -c 3 -o $O/pc python tools/ncu_c2.py 0 > $O/pc.log 2>&1
python tools/ncu_summary.py $O/pc.ncu-rep > $O/pc_summary.txt 2>&1
ncu -i $O/pc.ncu-rep --page source --csv --print-source sass > $O/pc_source.csv 2>/dev/null
rm -f $O/pc.ncu-rep
ls -la $O
