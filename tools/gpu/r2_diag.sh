# diagnosis of the 3-D reconstruction engines: DMMA throughput vs occupancy/ILP,
# per-phase cycle shares of engines 2 and 5 (config 3, 256^3), timing ablations
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench/dmma_occupancy.cu -o /tmp/dmma_occ && timeout 300 /tmp/dmma_occ > gpurun_out/dmma_occupancy.txt 2>&1
for e in 2 5; do
  KFVM_LIB=build/phase/libkfvm_b200.so timeout 300 python tools/phase_times.py 3 256 $e > gpurun_out/phase_e$e.txt 2>&1
done
out=gpurun_out/abl.txt; : > $out
timeout 300 python tools/time_step.py --config 3 >> $out 2>&1
timeout 300 python tools/time_step.py --config 3 --opt engine=2 >> $out 2>&1
for v in nophi noriemann nolimit; do
  KFVM_LIB=build/var_$v/libkfvm_b200.so timeout 300 python tools/time_step.py --config 3 >> $out 2>&1
done
cat $out
