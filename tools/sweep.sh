# BASELINE config sweep (north_star: per-kernel atom-steps/s on every named shape) + order sweep of config 4
# + the force-driver measurement (tools/bench_md.py).  Output: gpurun_out/sweep.jsonl, gpurun_out/md.jsonl
out=gpurun_out/sweep.jsonl; : > $out
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | tail -1 >> $out; }
for c in 1 2 3 5; do for m in ik ad; do run --config $c --mode $m; done; done
for s in 3 4 5 6 7; do for m in ik ad; do run --config 4 --order $s --mode $m; done; done
md=gpurun_out/md.jsonl; : > $md
for c in 2 4; do for p in fp64 mixed; do timeout 600 python tools/bench_md.py --config $c --precision $p 2>/dev/null | tail -1 >> $md; done; done
wc -l $out $md
