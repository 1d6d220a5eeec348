cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wide_engine.py tests/test_gpu_parity.py tests/test_gpu_parity_configs.py tests/test_boundaries.py tests/test_loopback.py -x -q -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_par.log
tail -6 gpurun_out/pytest_par.log
out=gpurun_out/bz.txt; : > $out
for rep in 1 2; do
for cfg in 3 4; do
  timeout 300 python tools/time_step.py --config $cfg --steps 3 >> $out 2>&1
  timeout 300 python tools/time_step.py --config $cfg --steps 3 --opt bounds_z=0 >> $out 2>&1
done
done
cat $out
