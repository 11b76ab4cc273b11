# Round-end evidence on one B200 (round 2): the GPU tests, every config's bench line, the
# reference arm, the ncu launch list of the default bench command, one full ncu capture of the
# timed wavefront launch and a range replay of the whole timed region (config 5).
set -x
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
for c in 5 4 2 3 1; do
  timeout 900 python bench.py --config $c > gpurun_out/r02/cfg$c.json 2> gpurun_out/r02/cfg$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/r02/reference_cfg5.json 2> gpurun_out/r02/reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02/launches_cfg5.csv python bench.py --steps 300 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r02/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wave_kernel -s 1 -c 1 -o gpurun_out/r02/wave_cfg5 python bench.py --steps 300 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r02/ncu_wave.log 2>&1; echo "ncu wave rc=$?"
SC_BENCH_NVTX=1 timeout 1800 ncu --replay-mode range --nvtx --nvtx-include bench_timed/ --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_active.avg,lts__t_bytes.sum -o gpurun_out/r02/range_cfg5 python bench.py --steps 300 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r02/ncu_range.log 2>&1; echo "ncu range rc=$?"
