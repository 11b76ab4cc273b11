set -e
python tools/quick_perf.py 2 > gpurun_out/qp.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fast_step_kernel -s 20 -c 1 -o gpurun_out/prof_fast python tools/quick_perf.py 2 > gpurun_out/ncu_log.txt 2>&1
echo done
