# Round-1 final-state measurement + profiles (run after the same commands exited 0 without ncu)
timeout 400 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttt > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sytrd_panel|sytrd_tail" -s 20 -c 2 \
  -o gpurun_out/sytrd_full python tools/eigbench.py 2000 > gpurun_out/ncu_full1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"EpiMvOff|EpiRowDot" -s 300 -c 2 -o gpurun_out/matvec_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ttt > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out
