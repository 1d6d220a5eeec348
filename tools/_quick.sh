cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu.log | head -5
for c in ${CONFIGS:-3}; do n=""; [ $c = 5 ] && n="--n 256"; [ $c = 4 ] && n="--n 256"; python bench.py --config $c $n --steps 3 --warmup 3 --no-cpu $BARGS 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c', '%.4e'%d['value'], d['roofline']['frac'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"; done
