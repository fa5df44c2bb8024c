set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -40
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-seconds 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
