for occ in 3 5 6; do
  echo "occ $occ"; RS_LIB=paper_2003_00575_b200/_lib/librangeseg_b200_occ$occ.so python bench.py --steps 20 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['plan'])"
done
echo "occ 4"; python bench.py --steps 20 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['plan'])"
echo "core"; python bench.py --steps 20 --no-cpu-baseline --no-e2e --core | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
for c in 2 3 4; do echo "config $c"; python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
