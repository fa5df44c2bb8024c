for v in "t256_o4 16" "t256_o4 8" "t384_o3 16" "t256_o3 16" "t256_o3 32"; do
  set -- $v
  echo "$1 rows=$2"; RS_LIB=paper_2003_00575_b200/_lib/librangeseg_b200_$1.so timeout 100 python bench.py --steps 50 --no-cpu-baseline --no-e2e --rows-per-cta $2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['plan'])" 2>&1 | tail -1
done
