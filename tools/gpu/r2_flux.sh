# ncu --set full of k_flux<3,2> and k_bounds<3> (config 3 at 256^3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_flux -s 1 -c 1 -o gpurun_out/prof_flux3 python tools/profile_step.py --config 3 --steps 1 > gpurun_out/ncu_flux3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bounds -s 1 -c 1 -o gpurun_out/prof_bounds3 python tools/profile_step.py --config 3 --steps 1 > gpurun_out/ncu_bounds3.log 2>&1
ls gpurun_out
