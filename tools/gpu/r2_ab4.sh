# A/B: mbarrier plane hand-off (no CTA barrier per plane) and the interleaved
# reciprocal batch in the weights phase, against build variants without each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_configs.py -x -q -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_par.log
out=gpurun_out/ab4.txt; : > $out
for v in "" $VARIANTS; do
  for cfg in 3 4; do
    if [ -z "$v" ]; then
      timeout 300 python tools/time_step.py --config $cfg --steps 3 >> $out 2>&1
    else
      KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py --config $cfg --steps 3 >> $out 2>&1
    fi
  done
done
timeout 300 python tools/time_step.py --config 3 --steps 3 >> $out 2>&1
timeout 300 python tools/time_step.py --config 4 --steps 3 >> $out 2>&1
cat $out; tail -3 gpurun_out/pytest_par.log
