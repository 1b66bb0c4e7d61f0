# A/B of library variants on config 5 (and config 3): bash tools/ab5.sh
A="--config 5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extra --no-config5"
run() { tag=$1; shift; env "$@" timeout 300 python bench.py $A > gpurun_out/ab5_$tag.json 2>gpurun_out/ab5_$tag.err; python -c "import json;d=json.loads(open('gpurun_out/ab5_$tag.json').readline());print('$tag',round(d['value']/1e9,3),{k:round(v*1e3,1) for k,v in d['phases_ms_per_step'].items()})" || tail -3 gpurun_out/ab5_$tag.err; }
run base X=1
for v in ${VARIANTS:-}; do run $v PPPM_B200_LIB=build/variants/$v/libpppm_b200.so; done
A="--steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-extra --no-config5"
run c3base X=1
