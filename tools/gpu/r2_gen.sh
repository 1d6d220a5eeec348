cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wide_engine.py tests/test_gpu_parity.py tests/test_boundaries.py tests/test_loopback.py -x -q -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_par.log
tail -12 gpurun_out/pytest_par.log
out=gpurun_out/gen.txt; : > $out
timeout 300 python tools/time_step.py --config 4 --n 200 --steps 3 >> $out 2>&1
timeout 300 python tools/time_step.py --config 4 --n 200 --steps 3 --opt wide=0 >> $out 2>&1
timeout 300 python tools/time_step.py --config 4 --steps 3 >> $out 2>&1
cat $out
