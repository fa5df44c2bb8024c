# A/B of two builds on the same box: default lib vs $1 (+ env variants), interleaved
L2=${1:-paper_2003_00575_b200/_lib/librangeseg_b200_ring.so}
for i in 1 2 3; do
  for v in "X=1" "RS_LIB=$L2 RS_NO_RING=1" "RS_LIB=$L2"; do
    printf "%-60s " "$v"
    env $v timeout 100 python bench.py --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))"
  done
done
