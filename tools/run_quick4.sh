timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/e2e_var.sh
