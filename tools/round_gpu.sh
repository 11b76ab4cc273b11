# Round-end evidence on one B200: GPU tests, the default bench line, the reference arm, the ncu
# launch list of the bench command and one full ncu capture of the step kernel.
set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fast_step_kernel -s 10 -c 1 -o gpurun_out/prof_cfg2 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fast_step_kernel -s 3 -c 1 -o gpurun_out/prof_cfg4 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/ncu_full4.log 2>&1; echo "ncu full4 rc=$?"
