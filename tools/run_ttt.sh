timeout 200 python tools/ttt_probe.py cfg1 tight 1e-6 2000
timeout 200 python tools/ttt_probe.py cfg2 paper 5e-3 2000
timeout 300 python tools/ttt_probe.py cfg5:0 tight 1e-6 1000
timeout 900 python tools/ttt_probe.py cfg3 tight 1e-6 1500
