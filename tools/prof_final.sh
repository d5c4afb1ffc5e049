# final-state measurement + profiles (each ncu command after the same command exited 0 without ncu)
timeout 400 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-ttt --steps 6 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --config cfg5 --batch 16 --max-iter 100 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttt > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sytrd_panel|sytrd_tail" -s 43 -c 2 \
  -o gpurun_out/eig_full python tools/eigbench.py 2000 > gpurun_out/ncu_full1.log 2>&1
ls -la gpurun_out | head -30
