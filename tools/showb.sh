for f in "$@"; do python -c "
import json,sys
try:
  d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'kernel', round(d['roofline']['kernel_ms'],3))
except Exception as e: print('$f', 'ERR', e)
"; done
