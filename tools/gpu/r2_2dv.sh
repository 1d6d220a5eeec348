cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/2dv.txt; : > $out
for rep in 1 2; do
  timeout 300 python bench.py --config 2 --no-cpu --steps 200 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('default', d['ms_per_step'], d['kernel_ms_per_step'])
" >> $out
  for v in $VARIANTS; do
    KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python bench.py --config 2 --no-cpu --steps 200 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', d['ms_per_step'], d['kernel_ms_per_step'])
" >> $out
  done
done
cat $out
