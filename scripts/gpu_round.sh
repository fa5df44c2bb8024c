# usage: bash scripts/gpu_round.sh TAG [ncu]
set -x
TAG=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
if [ "$2" = "ncu" ]; then
  python scripts/profile_one.py --batch 64 > gpurun_out/plain_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rs_fast -s 2 -c 1 -o gpurun_out/prof_$TAG python scripts/profile_one.py --batch 64 > gpurun_out/ncu_$TAG.log 2>&1
  echo ncu rc=$?
fi
