for rev in 0 1; do for hint in 0 1000000 100; do
  echo "rev=$rev hint=$hint"; SC_WAVE_REV=$rev SC_WAVE_HINT=$hint python tools/wave_perf.py --configs 5 --levels 12 --reps 2 2>&1 | grep wave
done; done
