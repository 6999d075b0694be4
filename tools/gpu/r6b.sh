# A/B: OPT-66B fc1 mid token counts with the K1 defaults vs the previous ones (QUIK_K1_STAGES=0 QUIK_K1_FILL=0)
for ab in new old new old; do
  if [ $ab = old ]; then export QUIK_K1_STAGES=0 QUIK_K1_FILL=0; else unset QUIK_K1_STAGES QUIK_K1_FILL; fi
  timeout 600 python tools/sweep.py --opt-m 256,1024,2048 --only "OPT-66B fc1" 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: continue
  print('$ab', r['name'], r['M'], round(r['step_ms']*1000,1), round(r['speedup_vs_f16'],2))"
done
