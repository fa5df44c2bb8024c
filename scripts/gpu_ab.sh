# A/B: env-var variants of the default bench (config 1 and 3)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in 1 3 2 4; do
for v in "" "RS_NO_RING=1"; do
  echo "=== config $cfg $v"
  env $v timeout 120 python bench.py --config $cfg --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
done; done
