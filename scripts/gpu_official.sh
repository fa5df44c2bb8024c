# Official measurement set: tests, bench line, launch list, full ncu of the bench workload.
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; echo ref rc=$?
cat gpurun_out/bench_ref_$TAG.json | tail -1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-cloud --no-per-config --no-check > gpurun_out/plain_launch_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rs_ -c 40 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-cloud --no-per-config --no-check > gpurun_out/ncu_launch_$TAG.log 2>&1
echo launches rc=$?
python scripts/profile_one.py --batch 256 > gpurun_out/plain_full_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rs_fast -s 2 -c 1 -o gpurun_out/full_$TAG python scripts/profile_one.py --batch 256 > gpurun_out/ncu_full_$TAG.log 2>&1
echo full rc=$?
