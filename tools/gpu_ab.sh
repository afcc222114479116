timeout 600 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/prof_workload.py raster c2 5
timeout 900 python bench.py --no-secondary --no-cpu-baseline > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; python -c "
import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['value'], d['e2e']['value'], d['phase_ms_per_step'])"
