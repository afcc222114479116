timeout 900 python bench.py > gpurun_out/bench1.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench1.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
timeout 900 python bench.py --steps 3 --warmup 3 --no-secondary > gpurun_out/bench1.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench1.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
