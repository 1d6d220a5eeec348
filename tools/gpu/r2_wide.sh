# the 16-warp W-cache engine (k_states_w) against k_states_u: parity, then timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_configs.py -x -q -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_par.log
tail -15 gpurun_out/pytest_par.log
out=gpurun_out/wide.txt; : > $out
for rep in 1 2; do
for cfg in 3 4; do
  timeout 300 python tools/time_step.py --config $cfg --steps 3 >> $out 2>&1
  timeout 300 python tools/time_step.py --config $cfg --steps 3 --opt wide=0 >> $out 2>&1
done
done
cat $out
