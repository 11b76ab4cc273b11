# Final evidence pass of the round on one B200: GPU tests, every bench line (default form and the
# driver's --steps 20 --warmup 5 form), the reference arm, ncu launch lists, range replays of the
# timed regions and full captures of the dominant kernels.
set -x
O=gpurun_out/final
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_active.avg,lts__t_bytes.sum
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
for c in 5 4 2 3 1; do
  timeout 900 python bench.py --config $c > $O/cfg$c.json 2> $O/cfg$c.err; echo "bench $c rc=$?"
done
for c in 5 4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/cfg${c}_s20.json 2> $O/cfg${c}_s20.err; echo "bench $c s20 rc=$?"
done
timeout 900 python bench.py --impl reference > $O/reference_cfg5.json 2> $O/reference.err; echo "ref rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/reference_cfg5_s20.json 2>> $O/reference.err; echo "ref s20 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_cfg5_s20.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > $O/ncu_list_s20.log 2>&1; echo "ncu list s20 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_cfg5.csv python bench.py --steps 300 --warmup 3 --no-cpu-baseline --e2e-calls 1 > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
SC_BENCH_NVTX=1 timeout 1500 ncu --replay-mode range --nvtx --nvtx-include bench_timed/ --clock-control none --metrics $M -f -o $O/range_cfg5_s20 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > $O/ncu_range5s.log 2>&1; echo "ncu range5 s20 rc=$?"
SC_BENCH_NVTX=1 timeout 1500 ncu --replay-mode range --nvtx --nvtx-include bench_timed/ --clock-control none --metrics $M -f -o $O/range_cfg4_s20 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > $O/ncu_range4s.log 2>&1; echo "ncu range4 s20 rc=$?"
SC_BENCH_NVTX=1 timeout 1800 ncu --replay-mode range --nvtx --nvtx-include bench_timed/ --clock-control none --metrics $M -f -o $O/range_cfg5 python bench.py --steps 300 --warmup 3 --no-cpu-baseline --e2e-calls 1 > $O/ncu_range5.log 2>&1; echo "ncu range5 rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fast_step_kernel -s 60 -c 1 -f -o $O/fast_cfg5_s20 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > $O/ncu_full5s.log 2>&1; echo "ncu full5 s20 rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wave_kernel -s 1 -c 1 -f -o $O/wave_cfg5 python bench.py --steps 300 --warmup 3 --no-cpu-baseline --e2e-calls 1 > $O/ncu_wave.log 2>&1; echo "ncu wave rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fast_step_kernel -s 10 -c 1 -f -o $O/step_cfg3 python bench.py --config 3 --steps 30 --warmup 3 --no-cpu-baseline --e2e-calls 1 > $O/ncu_cfg3.log 2>&1; echo "ncu cfg3 rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fast_step_kernel -s 5 -c 1 -f -o $O/step_cfg4 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 > $O/ncu_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"
for f in range_cfg5_s20 range_cfg4_s20 range_cfg5; do ncu -i $O/$f.ncu-rep --page raw --csv > $O/$f.csv 2>/dev/null; done
