cd $GRAFT_REPO_ROOT
CONFIGS="2 3" bash tools/gpu_check.sh
for ov in 1; do for c in 2 3; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu --opt overlap=$ov 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('overlap $ov cfg $c', '%.3e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
