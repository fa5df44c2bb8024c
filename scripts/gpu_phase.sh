mkdir -p gpurun_out
for args in "" "--core" "--skip 1" "--config 2" "--config 3" "--config 4 --core"; do
  echo "=== $args"; timeout 300 python scripts/phase_profile.py $args 2>&1 | tail -14
done
