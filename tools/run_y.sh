for e in "KOT_X=0" "KOT_COOP_YIELD=1" "KOT_X=0" "KOT_COOP_YIELD=1"; do echo "== $e"; env $e timeout 200 python bench.py --no-cpu-baseline --no-ttt 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); p=d['phases']
print('value %.3f e2e %.3f newton %.1f trial %.1f pipe_eg %.1f pipe_res %.1f wait %.1f' % (d['value'], d['e2e']['value'], p['host.newton']['ms_per_step'], p['host.trial_resid']['ms_per_step'], p['host.pipe_eg']['ms_per_step'], p['host.pipe_resid']['ms_per_step'], p['host.eg_wait']['ms_per_step']))"; done
