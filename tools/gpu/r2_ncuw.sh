cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_states_w -s 2 -c 1 -o gpurun_out/prof_c3_states_w python tools/profile_step.py --config 3 --steps 1 > gpurun_out/ncu_w.log 2>&1
tail -3 gpurun_out/ncu_w.log
