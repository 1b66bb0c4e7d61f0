for t in 0 1 0 1; do PPPM_B200_FIX64_TILES=$t timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-config5 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); x=d['extra']['fp64']; print('tiles $t fp64', round(x['value']/1e9,3), {k: round(v*1e3,1) for k,v in x['phases_ms_per_step'].items()})"; done
