set -x
mkdir -p gpurun_out
python scripts/profile_one.py --batch 64 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rs_segment -s 2 -c 1 -o gpurun_out/prof1 python scripts/profile_one.py --batch 64 > gpurun_out/ncu1.log 2>&1
echo rc=$?
tail -5 gpurun_out/ncu1.log
