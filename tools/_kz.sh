cd $GRAFT_REPO_ROOT
CONFIGS="2 3" bash tools/gpu_check.sh
for e in 3; do for kz in 8 16 32 64; do
python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --engine $e --kz $kz 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('engine $e kz $kz', '%.3e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
