mkdir -p gpurun_out/ab
for c in 3 2; do for i in 1 2; do timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-calls 1 > gpurun_out/ab/cfg${c}_$i.json 2>>gpurun_out/ab/err.txt; done; done
for c in 5 4; do for i in 1 2; do timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline --e2e-calls 1 > gpurun_out/ab/cfg${c}_s20_$i.json 2>>gpurun_out/ab/err.txt; done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab/cfg*.json')):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['steps'], '%.4e'%d['value'], round(d['ms_per_step']*1e3,2), 'e2e %.3e'%d['e2e']['value'])
PY
