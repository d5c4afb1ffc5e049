echo "== two-stage 2000"; KOT_EIG_STAGES=2 timeout 200 python tools/eigbench.py 2000 2>&1 | grep -v "^  Q:\|^  S:\|grid.sync"
echo "== one-stage 2000 grid 96"; KOT_TRD_GRID=96 timeout 200 python tools/eigbench.py 2000 2>&1 | head -14
