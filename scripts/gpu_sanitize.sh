# compute-sanitizer on the fused kernel: memcheck and synccheck on
# the default, S=1, mc14 and forced-overflow (node capacity 32) runs, racecheck
# (shared memory) on the default and the overflow path.  Logs in gpurun_out/sanitize_*.log.
mkdir -p gpurun_out
run() {  # name tool args...
  name=$1; tool=$2; shift 2
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python scripts/profile_one.py --iters 1 "$@" > gpurun_out/sanitize_${name}_${tool}.log 2>&1
  echo "$name $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${name}_${tool}.log | tail -1)"
}
for tool in memcheck synccheck; do
  run default $tool --batch 8 --check
  run S1 $tool --batch 8 --skip 1 --check
  run mc14 $tool --batch 4 --preset mc14 --check
  run overflow $tool --batch 4 --cap 32 --check
  run c3 $tool --config 3 --batch 16 --check
done
run default racecheck --batch 2
run overflow racecheck --batch 2 --cap 32
run S1 racecheck --batch 2 --skip 1
