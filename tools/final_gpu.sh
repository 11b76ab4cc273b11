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
# full captures: summarised on the box (tools/ncu_summary.py), the reports themselves stay there
# (gpurun brings back at most 64 MiB) except the wavefront one
full() {  # name, kernel regex, skip, node-updates per launch, title, bench args...
  local name=$1 rx=$2 skip=$3 nu=$4 title=$5; shift 5
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 -f -o $O/$name python bench.py "$@" --no-cpu-baseline --e2e-calls 1 > $O/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
  python tools/ncu_summary.py $O/$name.ncu-rep $nu "$title" $O/$name.txt > /dev/null 2>&1; echo "summary $name rc=$?"
}
full fast_cfg5_s20 fast_step_kernel 60 $((1024*128*128)) "r02 (final code, the driver's command form): one timed launch of fast_step_kernel on ONE of the four concurrent cloth chunks of config 5 (1024 cloths, whole-column units), captured alone (-k regex:fast_step_kernel -s 60 -c 1): the timed step runs four such launches at once (range replay: r02_range_bench_cfg5_s20.txt)" --steps 20 --warmup 5
rm -f $O/fast_cfg5_s20.ncu-rep
full step_cfg3 fast_step_kernel 10 $((1024*1024)) "r02 (final code): fast_step_kernel<ALPHA1, RING 4, GEN, ONLY_SPHERE, plain z> of bench.py --config 3, one timestep of the 1024^2 cloth (5-row single-warp units); -k regex:fast_step_kernel -s 10 -c 1" --config 3 --steps 30 --warmup 3
rm -f $O/step_cfg3.ncu-rep
full step_cfg4 fast_step_kernel 5 $((8192*8192)) "r02 (final code): fast_step_kernel (simple finish, wide-register) of bench.py --config 4, one timestep of the 8192^2 cloth; -k regex:fast_step_kernel -s 5 -c 1" --config 4 --steps 10 --warmup 3
rm -f $O/step_cfg4.ncu-rep
full wave_cfg5 wave_kernel 1 $((2731*128*128*300)) "r02 (final code): wave_kernel<ALPHA1, W=12, FIN=0> of bench.py --config 5, the timed launch (2731 collider-free cloths of 128^2 on 100 SMs, 300 timesteps; the plane cloths run concurrently in the streaming kernel, not under this capture); -k regex:wave_kernel -s 1 -c 1" --steps 300 --warmup 3
for f in range_cfg5_s20 range_cfg4_s20 range_cfg5; do ncu -i $O/$f.ncu-rep --page raw --csv > $O/$f.csv 2>/dev/null; rm -f $O/$f.ncu-rep; done
du -sh $O
