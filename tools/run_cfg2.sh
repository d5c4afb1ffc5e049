for e in "KOT_X=0" "KOT_TRD_TAIL=0" "KOT_MATVEC=full" "KOT_TRD_TAIL=0 KOT_MATVEC=full" "KOT_MATVEC=direct"; do
echo "== $e"; env $e timeout 200 python tools/ttt_probe.py cfg2 paper 5e-3 300 2>&1 | tail -1; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
