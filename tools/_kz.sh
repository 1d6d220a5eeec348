cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "kxrcf or engines or run_parity" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep -E "^E |FAILED" gpurun_out/pytest_gpu.log | head -5
for c in 3; do for kx in "" "--kxrcf"; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu $kx 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c $kx', '%.3e'%d['value'], d['kxrcf'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
