cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu.log | head -5
for rep in 1 2; do for t in 0 1; do
python bench.py --config 2 --steps 10 --warmup 3 --no-cpu --opt tma=$t 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tma $t', '%.4e'%d['value'], d['gpu_launches'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
