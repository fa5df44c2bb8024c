# usage: bash scripts/export_profiles.sh TAG  -- copy the official run's artefacts (gpurun_out/*_TAG.*) into profiles/r02
set -e
TAG=${1:-r02c}
D=profiles/r02
mkdir -p $D
cp gpurun_out/launches_$TAG.csv $D/launches_bench_config1.csv
cp gpurun_out/atomics_$TAG.csv $D/atomics_config1.csv
for n in c1 c2 S1; do
  ncu -i gpurun_out/full_${n}_$TAG.ncu-rep --page details --csv > $D/ncu_full_${n}_details.csv
  ncu -i gpurun_out/full_${n}_$TAG.ncu-rep --page raw --csv > $D/ncu_full_${n}_raw.csv
done
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_{tag}.json").read().strip().splitlines()[-1])
json.dump(d, open("profiles/r02/bench_line.json", "w"), indent=1)
r = json.loads(open(f"gpurun_out/bench_ref_{tag}.json").read().strip().splitlines()[-1])
json.dump(r, open("profiles/r02/bench_reference_line.json", "w"), indent=1)
PY
ls -la $D
