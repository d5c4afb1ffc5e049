for g in 36 48 64 148; do echo "== one-stage 2000 grid $g"; KOT_TRD_GRID=$g timeout 200 python tools/eigbench.py 2000 2>&1 | grep "sytrd_panel\|Q:\|S:\|sync"; done
