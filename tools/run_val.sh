timeout 200 python tools/ttt_probe.py cfg1 tight 1e-6 2000 2>&1 | tail -1
timeout 200 python tools/ttt_probe.py cfg2 tight 5e-3 300 2>&1 | tail -1
timeout 300 python tools/ttt_probe.py cfg5:0 tight 1e-6 1000 2>&1 | tail -1
timeout 300 python tools/ttt_probe.py cfg5:4 tight 1e-6 1000 2>&1 | tail -1
timeout 600 python bench.py --config cfg5 --batch 8 --max-iter 400 --profile tight 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('cfg5 tight batch8: problems/s %.3f converged %s iterations %s' % (d['value'], d['converged'], d['iterations']))"
