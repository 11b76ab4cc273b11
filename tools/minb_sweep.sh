for l in ab/libC.so ab/libD.so ab/libE.so; do echo "== $l"; SC_B200_LIB=$l python tools/sched_check.py 2 --seg=0,8,10,12,14,16,20,25; SC_B200_LIB=$l python tools/sched_check.py 4 5 3; done
