# one full ncu capture of the fast kernel on the headline workload (after a plain run)
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 120 python scripts/profile_one.py --batch 256 "$@" > gpurun_out/plain_full_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_fast -s 2 -c 1 -o gpurun_out/full_$TAG python scripts/profile_one.py --batch 256 "$@" > gpurun_out/ncu_full_$TAG.log 2>&1
echo full rc=$?
