cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-extra --no-cpu-baseline --no-alt 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_gpu_boundary.py -q -x -k "config4 or batched or stream or config1 or tiny or single_point or arccos or largest" 2>&1 | tail -3
