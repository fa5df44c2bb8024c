# Bounds-checked build (-DRS_CHECKED: every union-find node, listed edge, run
# id and cluster_sizes row is range-checked on the device and traps) under the
# GPU parity tests and the race-hunting stress fuzz.  compute-sanitizer is not
# available on this GPU pool (profiles/r02/sanitize_blocked.txt); this is the
# substitute.  Logs: gpurun_out/checked_*.log
mkdir -p gpurun_out
export RS_LIB=paper_2003_00575_b200/_lib/librangeseg_b200_checked.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contract.py tests/test_gpu_fuzz.py -m gpu -q -x \
  > gpurun_out/checked_tests.log 2>&1; echo "checked tests rc=$? $(tail -1 gpurun_out/checked_tests.log)"
timeout 900 python scripts/stress_fuzz.py 20 1 2 3 5 8 13 21:32 34:32 > gpurun_out/checked_stress.log 2>&1
echo "checked stress rc=$? $(tail -2 gpurun_out/checked_stress.log | tr '\n' ' ')"
