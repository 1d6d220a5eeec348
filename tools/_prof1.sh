cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flux -s 3 -c 1 -o gpurun_out/prof_flux22 python tools/profile_step.py --config 2 --steps 2 > gpurun_out/ncu2.log 2>&1; tail -2 gpurun_out/ncu2.log
