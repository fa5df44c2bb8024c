# variants: lib x rows_per_cta on config 1 (and 3)
for v in "librangeseg_b200 0" "librangeseg_b200_t1024_o1 64" "librangeseg_b200_t1024_o1 32" "librangeseg_b200_t768_o1 64"; do
  set -- $v
  for cfg in 1 3; do
    printf "%-28s rows=%-3s cfg=%s " $1 $2 $cfg
    RS_LIB=paper_2003_00575_b200/_lib/$1.so timeout 100 python bench.py --config $cfg --steps 50 --no-cpu-baseline --no-e2e --rows-per-cta $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), d['plan'])"
  done
done
