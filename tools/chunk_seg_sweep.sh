python tools/sched_check.py 2 5 --seg=0
SC_FAST_WIDE=1 python tools/sched_check.py 2 --seg=0
SC_FAST_WIDE=1 SC_CHUNK_SEG_ROWS=16 python tools/sched_check.py 2 --seg=0
SC_FAST_WIDE=1 SC_CHUNK_SEG_ROWS=10 python tools/sched_check.py 2 --seg=0
SC_CHUNKS=6 python tools/sched_check.py 2 --seg=0
SC_CHUNKS=2 python tools/sched_check.py 5 --seg=0
