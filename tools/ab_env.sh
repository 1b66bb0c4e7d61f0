# A/B of env settings on config 3: bash tools/ab_env.sh "name:VAR=1 VAR2=0" "name2:" ...  (each run twice, interleaved)
for spec in "$@" "$@"; do
name=${spec%%:*}; envs=${spec#*:}
env $envs timeout 120 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline ${MODEARG} > gpurun_out/ab_$name.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/ab_$name.json'));print('$name',round(d['value']/1e9,3),'G',{k:round(v*1e3,1) for k,v in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_$name.json
done
