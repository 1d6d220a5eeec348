# A/B of the current build against build variants ($VARIANTS) on the configs in $CFGS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_configs.py -x -q -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_par.log
out=gpurun_out/ab5.txt; : > $out
for rep in 1 2; do
for cfg in ${CFGS:-2 3 4}; do
  st=3; [ $cfg = 2 ] && st=50
  timeout 300 python tools/time_step.py --config $cfg --steps $st >> $out 2>&1
  for v in $VARIANTS; do
    KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py --config $cfg --steps $st >> $out 2>&1
  done
done
done
cat $out; tail -3 gpurun_out/pytest_par.log
