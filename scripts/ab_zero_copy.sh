python -m pytest tests/test_gpu_api.py tests/test_gpu_extras.py -m gpu -x -q -k "compact or host_session or prune or surgery" 2>&1 | tail -4
for z in 0 1 0 1; do SS_COMPACT_ZERO_COPY=$z python bench.py --steps 50 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=l['e2e']; print('zc=$z', round(l['value'],1), round(e['value'],1), round(e['stream_launched_value'],1), e['d2h_bytes_per_step'])"; done
