# A/B of library variants on config 3: bash tools/ab_lib.sh NAME... (build/variants/NAME; "main" = in-tree lib)
for v in "$@" "$@"; do
if [ "$v" = main ]; then L=""; else L="PPPM_B200_LIB=build/variants/$v/libpppm_b200.so"; fi
env $L timeout 120 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline ${MODEARG} > gpurun_out/ab_$v.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v',round(d['value']/1e9,3),'G',{k:round(v*1e3,1) for k,v in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_$v.json
done
