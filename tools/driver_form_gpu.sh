# Evidence for the command the driver runs (python bench.py --steps 20 --warmup 5): the bench
# line, the ncu launch list, a range replay of the whole timed region (config 5: 20 timesteps of
# the chunked streaming kernel, four concurrent cloth chunks) and one full capture of a timed
# streaming launch; the same range replay for config 4.
set -x
O=gpurun_out/r02d
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_active.avg,lts__t_bytes.sum
for i in 1 2 3; do
  timeout 900 python bench.py --steps 20 --warmup 5 > $O/cfg5_s20_run$i.json 2> $O/cfg5_s20_run$i.err; echo "bench rc=$?"
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/reference_s20.json 2> $O/reference_s20.err; echo "ref rc=$?"
timeout 900 python bench.py --config 4 --steps 20 --warmup 5 > $O/cfg4_s20.json 2> $O/cfg4_s20.err; echo "bench4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_cfg5_s20.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
SC_BENCH_NVTX=1 timeout 1500 ncu --replay-mode range --nvtx --nvtx-include bench_timed/ --clock-control none --metrics $M -o $O/range_cfg5_s20 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > $O/ncu_range5.log 2>&1; echo "ncu range5 rc=$?"
SC_BENCH_NVTX=1 timeout 1500 ncu --replay-mode range --nvtx --nvtx-include bench_timed/ --clock-control none --metrics $M -o $O/range_cfg4_s20 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > $O/ncu_range4.log 2>&1; echo "ncu range4 rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:fast_step_kernel -s 60 -c 1 -o $O/fast_cfg5_s20 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > $O/ncu_full5.log 2>&1; echo "ncu full5 rc=$?"
for f in range_cfg5_s20 range_cfg4_s20; do ncu -i $O/$f.ncu-rep --page raw --csv > $O/$f.csv 2>/dev/null; done
cat $O/cfg5_s20_run*.json | cut -c1-400
