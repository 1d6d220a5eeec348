# parity subset + step timing of the current build and of build variants
# (VARS: build/var_<name>), cases CASES (';'-separated time_step.py args)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -z "${NOTEST}" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_kxrcf.py tests/test_loopback.py tests/test_fused3.py ${TESTS} -x -q -p no:cacheprovider > gpurun_out/pytest_check.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_check.log
fi
out=gpurun_out/check.txt; : > $out
IFS=';' read -ra CS <<< "${CASES:---config 3;--config 4 --steps 2;--config 5 --n 256 --steps 2}"
for c in "${CS[@]}"; do
  echo "== $c" >> $out
  timeout 300 python tools/time_step.py $c >> $out 2>&1
  for v in ${VARS}; do
    KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py $c >> $out 2>&1
  done
done
tail -3 gpurun_out/pytest_check.log 2>/dev/null; cat $out
