cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in oldu new; do
KFVM_LIB=build/libkfvm_$v.so python bench.py --config 3 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
