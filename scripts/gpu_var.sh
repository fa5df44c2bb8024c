for v in "t512_o2 16" "t512_o2 32" "t1024_o1 32" "t1024_o1 64" "t256_o4 0"; do
  set -- $v
  echo "$1 rows=$2"; RS_LIB=paper_2003_00575_b200/_lib/librangeseg_b200_$1.so python bench.py --steps 50 --no-cpu-baseline --no-e2e --rows-per-cta $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['plan'])"
done
