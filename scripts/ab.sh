# Interleaved A/B of prebuilt libraries on the same box: bash scripts/ab.sh LIB1 LIB2 ... (config list via CFGS, extra bench args via ARGS)
CFGS=${CFGS:-"1 3"}
for cfg in $CFGS; do
  for i in 1 2 3; do
    for lib in "$@"; do
      printf "cfg %s %-45s " $cfg $(basename $lib)
      RS_LIB=$lib timeout 100 python bench.py --config $cfg --steps 60 --no-cpu-baseline --no-e2e --no-cloud --no-per-config --no-check $ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1))"
    done
  done
done
