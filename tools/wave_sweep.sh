# SC_WAVE_HINT sweep (sleep between mbarrier retries) on config 5 and a collider-free batch
for hint in 0 50 100 200 400 800; do
  echo "hint=$hint $(SC_WAVE_HINT=$hint timeout 100 python tools/cfg5_class_probe.py mixed simple-only 2>&1 | grep wave | tr '\n' ' ')"
done
