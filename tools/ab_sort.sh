# A/B of resident atom sorting on config 3 (env PPPM_B200_SORT_RESIDENT)
for s in 1 0 1 0; do
PPPM_B200_SORT_RESIDENT=$s timeout 120 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline ${MODEARG} > gpurun_out/ab_sort$s.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/ab_sort$s.json'));print('sort',$s,round(d['value']/1e9,3),'G',{k:round(v*1e3,1) for k,v in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_sort$s.json
done
