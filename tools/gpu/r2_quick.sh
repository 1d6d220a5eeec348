# quick check of the current build: fused-engine parity + config 3 step time
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fused3.py -x -q -p no:cacheprovider > gpurun_out/pytest_fused3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused3.log
out=gpurun_out/quick.txt; : > $out
timeout 300 python tools/time_step.py --config 3 >> $out 2>&1
timeout 300 python tools/time_step.py --config 3 --opt kz=64 >> $out 2>&1
for v in ${VARS:-}; do
  KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py --config 3 >> $out 2>&1
done
cat $out
