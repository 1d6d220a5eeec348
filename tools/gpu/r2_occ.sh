# occupancy sensitivity of engine 2 (3 vs 2 CTAs/SM) and the DMMA/DFMA interleave ubench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench/dmma_dfma_ratio.cu -o /tmp/ratio && timeout 120 /tmp/ratio > gpurun_out/dmma_dfma_ratio.txt 2>&1
out=gpurun_out/occ.txt; : > $out
timeout 300 python tools/time_step.py --config 3 >> $out 2>&1
KFVM_LIB=build/var_occ2/libkfvm_b200.so timeout 300 python tools/time_step.py --config 3 >> $out 2>&1
cat $out gpurun_out/dmma_dfma_ratio.txt
