# old/new A/B over configs: bash tools/ab_sweep.sh "ENV=VAL" "-"   (each argument one environment; "-" = defaults)
mkdir -p gpurun_out
run() { env $E timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-config5 --no-extra "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$E', '$*', round(d['value']/1e9,3), {k: round(v*1e3,1) for k,v in d['phases_ms_per_step'].items()})" ; }
for e in "$@"; do
  if [ "$e" = "-" ]; then E=""; else E="$e"; fi
  run --config 3 --mode ad
  run --config 5 --mode ik
  for s in 3 4 5 6 7; do run --config 4 --order $s --mode ik; done
  env $E timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-config5 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); x=d['extra']; print('$E', 'c3', round(d['value']/1e9,3), 'md', round(x['md']['value']/1e9,3), {k: round(v*1e3,1) for k,v in x['md']['phases_ms_per_step'].items()}, 'binned', round(x['binned']['value']/1e9,3))"
done
