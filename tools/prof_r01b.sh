# Round-1 (session 2) measurement + profiles: bench lines, ncu launch list, ncu full captures.
timeout 400 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-ttt --steps 6 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttt > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sytrd_panel" -s 40 -c 1 \
  -o gpurun_out/sytrd_full python tools/eigbench.py 2000 > gpurun_out/ncu_full1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"EpiMvOff|EpiRowDot" -s 400 -c 2 \
  -o gpurun_out/matvec_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-ttt > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out
