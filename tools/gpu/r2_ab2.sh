# A/B of build variants (VARS) on both 3-D engines, config 3 (256^3) and config 4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/ab2.txt; : > $out
for cfg in ${CFGS:-3}; do
for e in 2 5; do
  echo "== config $cfg engine $e" >> $out
  timeout 300 python tools/time_step.py --config $cfg --opt engine=$e >> $out 2>&1
  for v in ${VARS}; do
    KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py --config $cfg --opt engine=$e >> $out 2>&1
  done
done
done
cat $out
