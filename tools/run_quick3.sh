timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/e2e_var.sh
timeout 400 python bench.py --config cfg5 --batch 16 --max-iter 100 2>&1 | tail -1 | cut -c1-200
KOT_TRD_GRID=48 timeout 300 python tools/conc_probe.py 8 40 4 2>&1 | tail -1
