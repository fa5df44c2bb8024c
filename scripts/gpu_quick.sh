# quick GPU iteration: parity tests, short bench on the headline + other configs, ablation
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for args in "" "--config 2" "--config 3" "--config 4" "--skip 1" "--core"; do
  echo "=== bench $args"
  timeout 120 python bench.py --steps 50 --no-cpu-baseline --no-e2e $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
timeout 120 python scripts/ablation.py 1 2>&1 | tail -14
