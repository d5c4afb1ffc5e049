timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sytrd_tail" -c 1 \
  -o gpurun_out/tail_full python tools/eigbench.py 1000 > gpurun_out/ncu_tail.log 2>&1
ncu -i gpurun_out/tail_full.ncu-rep --page source --csv > gpurun_out/tail_source.csv 2>/dev/null
ls -la gpurun_out/tail*
