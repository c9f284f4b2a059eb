# e2e per-call time with the process pinned to single vCPUs (host placement check)
for c in 0 3 7 8 11 15 none none; do
  if [ "$c" = none ]; then pre=""; else pre="taskset -c $c"; fi
  $pre python tools/e2e_spread.py 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$c', d['mode'], round(d['mean_ms'],3), round(d['median_ms'],3))"
done
