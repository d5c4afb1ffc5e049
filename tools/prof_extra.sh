timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"1, 2, EpiRowDot|EpiMvOff" -s 40 -c 2 -o gpurun_out/matvec_full3 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ttt > gpurun_out/ncu_mv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"q2_wave" -c 1 \
  -o gpurun_out/q2_full python tools/eigbench.py 4096 > gpurun_out/ncu_q2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sb2st" -c 1 \
  -o gpurun_out/sb2st_full python tools/eigbench.py 4096 > gpurun_out/ncu_sb.log 2>&1
ls -la gpurun_out/*.ncu-rep
