mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "sym_eig or eg_step or lockstep or tridiagonal" > gpurun_out/pytest_eig.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_eig.log
timeout 200 python tools/eigbench.py 2000 > gpurun_out/eigbench2000_b.txt 2>&1
timeout 300 python tools/setup_probe.py > gpurun_out/setup_probe.txt 2>&1
CUDA_MODULE_LOADING=EAGER timeout 300 python tools/setup_probe.py > gpurun_out/setup_probe_eager.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-batch --no-ttt > gpurun_out/bench_nb.json 2> gpurun_out/bench_nb.err
