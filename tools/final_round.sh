timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_final.log
timeout 400 python bench.py > gpurun_out/bench_cfg3_final.json 2> gpurun_out/bench_cfg3_final.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-ttt --steps 6 > gpurun_out/bench_cfg4_final.json 2> gpurun_out/bench_cfg4_final.err
timeout 600 python bench.py --config cfg5 --batch 16 --max-iter 100 > gpurun_out/bench_cfg5_final.json 2> gpurun_out/bench_cfg5_final.err
timeout 300 python tools/eigbench.py 2000 > gpurun_out/eigbench2000_final.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_bench_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttt > gpurun_out/ncu_launch_final.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sytrd_panel|sytrd_tail" -s 43 -c 2 -o gpurun_out/eig_full_final python tools/eigbench.py 2000 > gpurun_out/ncu_full_final.log 2>&1
ls gpurun_out
