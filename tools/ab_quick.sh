# quick A/B on config 3: bash tools/ab_quick.sh "ENV=VAL ..." "ENV=VAL ..." (each argument one environment; "-" = defaults)
mkdir -p gpurun_out
i=0
for e in "$@" "$@"; do
  i=$((i+1))
  if [ "$e" = "-" ]; then E=""; else E="$e"; fi
  env $E timeout 200 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-config5 ${ABARGS:---no-extra} > gpurun_out/abq_$i.json 2> gpurun_out/abq_$i.err
  python - "$e" gpurun_out/abq_$i.json <<'P'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    x = d.get('extra', {})
    print(sys.argv[1], round(d['value'] / 1e9, 3), 'G', {k: round(v * 1e3, 1) for k, v in d['phases_ms_per_step'].items()},
          'md', round(x.get('md', {}).get('value', 0) / 1e9, 3), {k: round(v * 1e3, 1) for k, v in x.get('md', {}).get('phases_ms_per_step', {}).items()},
          d['clocks']['sm_mhz'])
except Exception as ex:
    print(sys.argv[1], 'failed', ex)
P
done
