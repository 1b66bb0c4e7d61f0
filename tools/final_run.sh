# Round artifacts on one B200 (run under gpurun from the repo root):
#   GPU tests, smoke, bench line + reference arm, config/order sweep + force driver,
#   ncu launch list and --set full captures of the top kernels -> gpurun_out/
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 300 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench.err; echo "bench=$?"
timeout 300 python bench.py --impl reference > gpurun_out/bench_r01_ref.json 2> gpurun_out/bench_ref.err; echo "ref=$?"
bash tools/sweep.sh > gpurun_out/sweep.log 2>&1; echo "sweep=$?"
A="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 120 python bench.py $A > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/launches_r01.csv python bench.py $A > gpurun_out/ncu_launch.log 2>&1; echo "launches=$?"
for k in k_gather_ws k_spread_tma k_zfft_green k_plane_c2r; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/r01_full_$k \
    python bench.py $A > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k=$?"
done
PPPM_B200_GATHER=4 timeout 120 python bench.py $A > /dev/null 2>&1 && PPPM_B200_GATHER=4 timeout 300 ncu --set full \
  --clock-control none --import-source on -k regex:k_gather_mma -s 1 -c 1 -o gpurun_out/r01_full_k_gather_mma \
  python bench.py $A > gpurun_out/ncu_mma.log 2>&1; echo "ncu mma=$?"
# the multi-GPU (z-slab, NCCL) code path end to end with one slab
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --force-slab --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/slab1.json 2> gpurun_out/slab1.err
echo "slab=$?"
