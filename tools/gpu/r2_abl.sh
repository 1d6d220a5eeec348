# timing ablations of the fused 3-D engine (config 3, 256^3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/abl.txt; : > $out
timeout 300 python tools/time_step.py --config 3 >> $out 2>&1
for v in nophi noriemann nolimit nobeta notail minb2; do
  KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py --config 3 >> $out 2>&1
done
timeout 300 python tools/time_step.py --config 3 --opt engine=2 >> $out 2>&1
cat $out
