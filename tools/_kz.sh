cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "flux_kernels" 2>&1 | tail -2
for c in 2 3; do for fc in 0 1; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu --opt flux_cp=$fc 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c fc $fc', '%.4e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
