# A/B of the fp32 kernel variants on config 3 (env: PPPM_B200_SPREAD / PPPM_B200_GATHER)
for v in "1 1" "3 1" "1 0" "0 1"; do set -- $v
PPPM_B200_SPREAD=$1 PPPM_B200_GATHER=$2 timeout 120 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline ${MODEARG} > gpurun_out/ab_$1$2.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/ab_$1$2.json'));print('spread',$1,'gather',$2,round(d['value']/1e9,3),'G',{k:round(v*1e3,1) for k,v in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
done
