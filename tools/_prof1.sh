cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_states_row -s 3 -c 1 -o gpurun_out/prof_row22 python tools/profile_step.py --config 2 --steps 2 --engine 3 > gpurun_out/ncu1.log 2>&1; tail -2 gpurun_out/ncu1.log
