# profile the fused 3-D engine: per-phase cycle counters and one ncu --set full
# capture of k_fused3 (config 3 recipe at 128^3 / 256^3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=${N:-128}
KFVM_LIB=build/phase/libkfvm_b200.so timeout 300 python tools/phase_times.py 3 $N 5 > gpurun_out/phase_fused3.txt 2>&1
KFVM_LIB=build/phase/libkfvm_b200.so timeout 300 python tools/phase_times.py 3 $N 2 > gpurun_out/phase_u.txt 2>&1
rm -f gpurun_out/prof_fused3.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused3 -s 2 -c 1 -o gpurun_out/prof_fused3 python tools/profile_step.py --config 3 --n $N --steps 1 > gpurun_out/ncu_fused3.log 2>&1
ls -la gpurun_out
