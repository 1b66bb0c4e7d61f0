# Round artifacts on one B200 (run under gpurun from the repo root):
#   bash tools/final_run.sh TAG
# GPU tests, smoke, bench line + reference arm, config/order sweep + force driver,
# reference suite (fp64 / mixed), ncu launch lists (config 3, config 5) and
# --set full captures of the top kernels -> gpurun_out/
set -u
T=${1:-r02}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest=$?"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke=$?"
timeout 600 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_${T}_ref.json 2> gpurun_out/bench_ref_$T.err; echo "ref=$?"
for p in fp64 mixed; do
  timeout 600 python tests/run_reference_suite.py --precision $p --out gpurun_out/refsuite_${T}_$p.json > gpurun_out/refsuite_${T}_$p.log 2>&1
  echo "refsuite $p=$?"
done
bash tools/sweep.sh > gpurun_out/sweep.log 2>&1; echo "sweep=$?"
timeout 600 python tools/density_probe.py > gpurun_out/density_$T.jsonl 2>&1; echo "density=$?"
A="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-config5 --no-extra"
timeout 120 python bench.py $A > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/launches_$T.csv python bench.py $A > gpurun_out/ncu_launch.log 2>&1; echo "launches=$?"
B="--config 5 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-extra --no-config5"
timeout 300 python bench.py $B > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_${T}_config5.csv python bench.py $B > gpurun_out/ncu_launch5.log 2>&1; echo "launches5=$?"
for k in k_gather_ws k_spread_res k_zfft_green k_plane_c2r; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/${T}_full_$k \
    python bench.py $A > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k=$?"
done
