# Official measurement set: GPU tests, bench line, reference arm, launch list,
# ncu --set full captures (config 1, config 2, S=1) and union-find atomic metrics.
# Each ncu pass runs after the same command has exited 0 without ncu.
set -x
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_ref_$TAG.json 2>&1; echo ref rc=$?
tail -c 400 gpurun_out/bench_ref_$TAG.json
Q="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-cloud --no-per-config --no-check --no-frame-api"
python bench.py $Q > gpurun_out/plain_launch_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rs_ -c 40 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py $Q > gpurun_out/ncu_launch_$TAG.log 2>&1
echo launches rc=$?
for spec in "c1:--config 1" "c2:--config 2" "S1:--config 1 --skip 1"; do
  name=${spec%%:*}; args=${spec#*:}
  python scripts/profile_one.py --batch 256 $args > gpurun_out/plain_full_${name}_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rs_fast -s 2 -c 1 -o gpurun_out/full_${name}_$TAG python scripts/profile_one.py --batch 256 $args > gpurun_out/ncu_full_${name}_$TAG.log 2>&1
  echo full $name rc=$?
done
ncu --clock-control none -k regex:rs_fast -s 2 -c 1 --csv --metrics \
gpu__time_duration.sum,smsp__inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__t_bytes_pipe_lsu_mem_dshared_op_atom.sum,lts__t_sectors_srcunit_tex_op_atom.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  python scripts/profile_one.py --batch 256 > gpurun_out/atomics_$TAG.csv 2>&1
echo atomics rc=$?
