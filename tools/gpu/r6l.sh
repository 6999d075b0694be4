for i in 1 2 3; do
timeout 600 python tools/sweep.py --only "cfg2 7B down" 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: continue
  print(r['name'], r['M'], round(r['step_ms']*1000,1), round(r['speedup_vs_f16'],2))"
timeout 600 python tools/sweep.py --only "13B" 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: continue
  print(r['name'], r['M'], round(r['step_ms']*1000,1), round(r['speedup_vs_f16'],2))"
done
