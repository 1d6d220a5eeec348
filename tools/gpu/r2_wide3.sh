cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/wide3.txt; : > $out
for cfg in 3 4; do
  for v in $VARIANTS; do
    echo "-- $v" >> $out
    KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py --config $cfg --steps 3 >> $out 2>&1
    KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py --config $cfg --steps 3 --opt kz=64 >> $out 2>&1
  done
done
KFVM_LIB=build/var_wskew6/libkfvm_b200.so timeout 300 python tools/time_step.py --config 4 --steps 3 --opt kz=16 >> $out 2>&1
KFVM_LIB=build/var_wskew6/libkfvm_b200.so timeout 300 python tools/time_step.py --config 4 --steps 3 --opt kz=128 >> $out 2>&1
cat $out
