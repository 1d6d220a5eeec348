# A/B timing of build variants and options on the fused 3-D engine
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fused3.py -x -q -p no:cacheprovider > gpurun_out/pytest_fused3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused3.log
out=gpurun_out/ab.txt; : > $out
run() {  # label, env, args
  echo "== $1" >> $out
  env $2 timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 $3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value %.4g frac %.4f whole %.4f' % (d['value'], d['roofline']['frac'], d['whole_step_fp64_frac']), d['kernel_ms_per_step'], d['clocks']['reasons'])
    elif 'Error' in l or 'error' in l: print(l.strip())
" >> $out
}
for cfg in 3 4; do
  run "cfg$cfg default" "" "--config $cfg"
  run "cfg$cfg minb2" "KFVM_LIB=build/var_minb2/libkfvm_b200.so" "--config $cfg"
  run "cfg$cfg kz16" "" "--config $cfg --kz 16"
  run "cfg$cfg kz64" "" "--config $cfg --kz 64"
  run "cfg$cfg engine2" "" "--config $cfg --engine 2"
done
KFVM_LIB=build/phase/libkfvm_b200.so timeout 300 python tools/phase_times.py 3 128 5 > gpurun_out/phase_fused3.txt 2>&1
cat $out
