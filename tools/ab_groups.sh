# e2e (PppmContext.compute through pppm_compute_ex, host buffers) against the atom groups:
#   bash tools/ab_groups.sh G:LAST ...   (PPPM_B200_GROUPS : PPPM_B200_GROUP_LAST)
for a in "$@"; do
g=${a%%:*}; l=${a##*:}
PPPM_B200_GROUPS=$g PPPM_B200_GROUP_LAST=$l timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-config5 --no-extra > gpurun_out/grp_$g.json 2> gpurun_out/grp_$g.err
python -c "
import json
d=json.loads([l for l in open('gpurun_out/grp_$g.json') if l.startswith('{')][-1])
print('groups $g last $l', 'e2e', round(d['e2e']['value']/1e9,3), 'f64', round(d['e2e']['value_f64_forces']/1e9,3), 'value', round(d['value']/1e9,3))" || tail -3 gpurun_out/grp_$g.err
done
