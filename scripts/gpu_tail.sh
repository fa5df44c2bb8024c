# Wave-quantisation experiment: batch scaling, split launches, and band /
# CTA-size variants (prebuilt libraries from build_flags_variant.sh).
mkdir -p gpurun_out
L=paper_2003_00575_b200/_lib
b() {  # lib rows cfg
  printf "%-28s rows %-3s cfg %s  " "$(basename $1)" "$2" "$3"
  RS_LIB=$1 timeout 120 python bench.py --config $3 --rows-per-cta $2 --steps 60 --no-cpu-baseline --no-e2e --no-cloud 2>&1 \
    | python -c "import json,sys; t=sys.stdin.read(); d=json.loads(t.strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1))" 2>&1 | tail -1
}
timeout 300 python scripts/tail_exp.py
for cfg in 1 2 3 4; do
  for v in "$L/librangeseg_b200.so 0" "$L/librangeseg_b200.so 16" "$L/librangeseg_b200_t256o4.so 16" \
           "$L/librangeseg_b200_t256o4.so 8" "$L/librangeseg_b200_t1024o1.so 0"; do
    set -- $v; b $1 $2 $cfg
  done
done
