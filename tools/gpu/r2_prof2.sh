# phase counters + ncu --set full of the tensor engine (config 3 at 128^3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
KFVM_LIB=build/phase/libkfvm_b200.so timeout 300 python tools/phase_times.py 3 256 2 > gpurun_out/phase_e2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_states_u -s 2 -c 1 -o gpurun_out/prof_e2b python tools/profile_step.py --config 3 --n 128 --engine 2 > gpurun_out/ncu_e2b.log 2>&1
cat gpurun_out/phase_e2.txt
