cd $GRAFT_REPO_ROOT
KFVM_LIB=build/libkfvm_ws4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "engines" 2>&1 | tail -2
for mb in 3 4; do for kz in 8 16 32; do
KFVM_LIB=build/libkfvm_ws$mb.so python bench.py --config 2 --steps 10 --warmup 3 --no-cpu --engine 5 --kz $kz 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ws minb $mb kz $kz', '%.4e'%d['value'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
