# A/B of build variants (VARS) on engine 2: configs 3, 4 and the config 5 recipe at 256^3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/ab3.txt; : > $out
for c in "--config 3" "--config 4 --steps 2" "--config 5 --n 256 --steps 2"; do
  echo "== $c" >> $out
  timeout 300 python tools/time_step.py $c --opt engine=2 >> $out 2>&1
  for v in ${VARS}; do
    KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py $c --opt engine=2 >> $out 2>&1
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_fused3.py -x -q -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
cat $out; tail -3 gpurun_out/pytest_quick.log
