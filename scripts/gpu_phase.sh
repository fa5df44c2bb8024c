mkdir -p gpurun_out
for args in "" "--core" "--skip 1" "--config 2" "--config 2 --skip 1" "--config 3" "--config 4" "--config 4 --skip 1"; do
  echo "=== $args"; timeout 300 python scripts/phase_profile.py $args 2>&1 | tail -44
done
