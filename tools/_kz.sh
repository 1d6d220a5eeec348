cd $GRAFT_REPO_ROOT
for kz in 1 2 4 8; do
python bench.py --config 2 --steps 10 --warmup 3 --no-cpu --opt flux_update=1 --opt flux_update_kz=$kz 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kz $kz', '%.4e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done
