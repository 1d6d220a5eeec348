cd $GRAFT_REPO_ROOT
for v in 2_49152 3_0 3_49152; do for kz in 8 16; do
KFVM_LIB=build/libkfvm_u$v.so python bench.py --config 3 --n 192 --steps 3 --warmup 3 --no-cpu --kz $kz 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('u $v kz $kz', '%.3e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
