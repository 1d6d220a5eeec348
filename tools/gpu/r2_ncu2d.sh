cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_row -s 6 -c 1 -o gpurun_out/prof_c2_states python tools/profile_step.py --config 2 --steps 3 > gpurun_out/ncu_2d.log 2>&1
tail -2 gpurun_out/ncu_2d.log
