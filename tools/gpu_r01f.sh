# GPU pass: parity tests incl. Spearman, one-rank NCCL bench with population sharding.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 MASTER_ADDR=127.0.0.1 MASTER_PORT=29511 timeout 600 python bench.py --nccl --shard programs --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_progshard.log 2>&1; tail -1 gpurun_out/bench_c3_progshard.log > gpurun_out/bench_r01_v12_c3_nccl_programs.json
