cd $GRAFT_REPO_ROOT
for mb in 6 7 8; do for kz in 4 8; do
KFVM_LIB=build/libkfvm_r$mb.so python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --engine 4 --kz $kz 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb $mb kz $kz engine 4', '%.3e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
