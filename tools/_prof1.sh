cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_states_u -s 3 -c 1 -o gpurun_out/prof_u32b python tools/profile_step.py --config 3 --n 128 --steps 2 > gpurun_out/ncu1.log 2>&1; tail -1 gpurun_out/ncu1.log
