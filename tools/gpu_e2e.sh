cd $GRAFT_REPO_ROOT
free -g | head -2
timeout 900 python -m pytest tests -x -q -m gpu -k "batch or host_path" 2>&1 | tail -3
for k in 3 6; do timeout 900 python bench.py --steps $k --warmup 3 --no-also --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('steps', d['steps'], 'value', round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks'])"; done
