cd $GRAFT_REPO_ROOT
for mb in 1 6 8; do for c in 2 3; do
KFVM_LIB=build/libkfvm_fl$mb.so python bench.py --config $c --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('flux minb $mb cfg $c', '%.3e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
