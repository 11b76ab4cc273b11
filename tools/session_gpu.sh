mkdir -p gpurun_out/s4
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
for c in 5 4 2 3 1; do
  timeout 900 python bench.py --config $c > gpurun_out/s4/cfg$c.json 2> gpurun_out/s4/cfg$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/s4/reference_cfg5.json 2> gpurun_out/s4/reference.err; echo "ref rc=$?"
tail -3 gpurun_out/s4/pytest_gpu.txt; cat gpurun_out/s4/cfg*.json
