# ncu --set full captures (source-level) of the two 3-D engines on config 3 at 128^3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_states_u -s 2 -c 1 -o gpurun_out/prof_e2 python tools/profile_step.py --config 3 --n 128 --engine 2 > gpurun_out/ncu_e2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused3 -s 2 -c 1 -o gpurun_out/prof_e5 python tools/profile_step.py --config 3 --n 128 --engine 5 > gpurun_out/ncu_e5.log 2>&1
ls -la gpurun_out
