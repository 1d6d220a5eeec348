cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu.log | head -5
python bench.py --config 3 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', '%.4e'%d['value'], d['roofline']['frac'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
python bench.py --config 5 --n 256 --steps 2 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5@256', '%.4e'%d['value'], d['roofline']['frac'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
python bench.py --config 4 --n 256 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4@256', '%.4e'%d['value'], d['roofline']['frac'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
