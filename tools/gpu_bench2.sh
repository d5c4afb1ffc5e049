# bench (default) + cfg5 probe at the paper threshold
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "rc=$?" >> gpurun_out/bench_default.err
timeout 600 python bench.py --config cfg5 --batch 32 --max-iter 100 --tol 5e-3 --profile tight > gpurun_out/bench_cfg5_probe.json 2> gpurun_out/bench_cfg5_probe.err; echo "rc=$?" >> gpurun_out/bench_cfg5_probe.err
