mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "row_sharded or two_process or middle_operator or lockstep" > gpurun_out/pytest_shard.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shard.log
