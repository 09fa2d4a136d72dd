for m in off off off nvml nvml nvml smi smi; do SD_BENCH_CLOCKS=$m timeout 300 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$m', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['clocks'])"; done
