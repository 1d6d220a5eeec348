cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_configs.py tests/test_kxrcf.py -x -q -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_par.log
tail -12 gpurun_out/pytest_par.log
out=gpurun_out/r3.txt; : > $out
for rep in 1 2; do
  timeout 300 python tools/time_step.py --config 5 --n 256 --steps 2 >> $out 2>&1
  for v in $VARIANTS; do
    KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py --config 5 --n 256 --steps 2 >> $out 2>&1
  done
done
cat $out
