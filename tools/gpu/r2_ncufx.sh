cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flux -s 1 -c 1 -o gpurun_out/prof_c3_flux python tools/profile_step.py --config 3 --steps 1 > gpurun_out/ncu_fx.log 2>&1
tail -2 gpurun_out/ncu_fx.log
