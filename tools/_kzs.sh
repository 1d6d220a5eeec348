cd $GRAFT_REPO_ROOT
for kz in ${KZS:-8 12 16 24 32}; do python bench.py --config ${CFG:-3} $NARG --steps 3 --warmup 3 --no-cpu --kz $kz 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kz $kz', '%.4e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"; done
