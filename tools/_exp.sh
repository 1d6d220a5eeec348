# A/B of compile-time variants on the GPU box: EXPS = ;-separated EXTRA flag
# sets, CFGS = configs to bench per variant.
cd $GRAFT_REPO_ROOT
b() { python bench.py --config $1 --steps ${STEPS:-3} --warmup 3 --no-cpu $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2 cfg $1', '%.4e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})" 2>&1 | tail -1; }
echo "${EXPS:-}" | tr ';' '\n' | while read -r e; do
make -B EXTRA="$e" -j8 > gpurun_out/make_exp.log 2>&1 || tail gpurun_out/make_exp.log
for c in ${CFGS:-2 3}; do b $c "$e" "$BARGS"; done
done
