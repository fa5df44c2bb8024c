for b in 64 148 256; do echo "=== batch $b"; timeout 120 python scripts/phase_profile.py --batch $b 2>&1 | tail -21; done
