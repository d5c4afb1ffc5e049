timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/e2e_var.sh 2>&1 | head -4
timeout 200 python tools/ttt_probe.py cfg5:0 tight 1e-6 1000 2>&1 | tail -1
