# A/B of kernel variants / graphs on config 3 (env: PPPM_B200_SPREAD / PPPM_B200_GATHER / PPPM_B200_GRAPHS)
for v in "1 1 1" "1 1 0" "1 0 1"; do set -- $v
PPPM_B200_SPREAD=$1 PPPM_B200_GATHER=$2 PPPM_B200_GRAPHS=$3 timeout 120 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline ${MODEARG} > gpurun_out/ab_$1$2$3.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/ab_$1$2$3.json'));print('spread',$1,'gather',$2,'graphs',$3,round(d['value']/1e9,3),'G',{k:round(v*1e3,1) for k,v in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_$1$2$3.json
done
