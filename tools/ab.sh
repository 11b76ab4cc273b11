# usage: bash tools/ab.sh "<cfgs>"  — A/B device time: ab/libA.so vs the in-tree library, alternated
for i in 1 2; do
  echo "A:"; SC_B200_LIB=ab/libA.so python tools/sched_check.py $1
  echo "B:"; python tools/sched_check.py $1
done
