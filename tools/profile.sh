# round-2 profiles (each ncu command right after the same command exited 0 without ncu)
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttt --no-batch"
$B > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/launches_bench_r02.csv \
  $B > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/eigbench.py 2000 > gpurun_out/plain_eig.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
  -k regex:"sytrd_panel" -s 43 -c 43 --csv --log-file gpurun_out/panel_traffic_r02.csv python tools/eigbench.py 2000 > gpurun_out/ncu_panel.log 2>&1
echo "panel traffic rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sytrd_panel|sytrd_tail" -s 64 -c 2 \
  -o gpurun_out/eig_full_r02 python tools/eigbench.py 2000 > gpurun_out/ncu_eig_full.log 2>&1
echo "eig full rc=$?"
$B > gpurun_out/plain_bench2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm_tma_kernel.*(EpiMvOff|EpiRowDot)" -s 40 -c 4 -o gpurun_out/gemm_full_r02 $B > gpurun_out/ncu_gemm_full.log 2>&1
echo "gemm full rc=$?"
ls -la gpurun_out
