# FAST stepping in K concurrent cloth chunks (capi.cu chunked_fast_steps): device time per K
for k in 0 2 3 4 6 8 12 16; do echo "K=$k"; SC_CHUNKS=$k python tools/sched_check.py 2 5; done
