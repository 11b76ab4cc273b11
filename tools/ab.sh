# usage: bash tools/ab.sh "<cfgs>" [libs...] — alternated device timing of library builds
# (default: ab/libA.so vs the in-tree library)
cfgs=$1; shift
libs=${@:-ab/libA.so tree}
for i in 1 2; do
  for l in $libs; do
    echo "$l:"
    if [ "$l" = tree ]; then python tools/sched_check.py $cfgs; else SC_B200_LIB=$l python tools/sched_check.py $cfgs; fi
  done
done
