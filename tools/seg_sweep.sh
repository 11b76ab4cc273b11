for sr in 4 5 6 7 8 10 12 15 19 22; do echo -n "seg=$sr "; SC_FAST_SEG_ROWS=$sr python tools/sched_check.py 2 --seg=$sr; done
for sr in 28 40 55 64 80 110; do echo -n "seg=$sr "; SC_FAST_SEG_ROWS=$sr python tools/sched_check.py 4 --seg=$sr; done
