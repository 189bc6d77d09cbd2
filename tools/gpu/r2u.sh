export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fast.py tests/test_gpu_skew.py tests/test_gpu_qr_paths.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'ttmctc', d['ttmctc']['value'], d['ttmctc']['per_mode_ms'], 'e2e', d['e2e']['value'])"
